# C2 bench line, one-GPU projections of the row-sharded runs, maturity sweep
set -x
timeout 900 python bench.py --config c2 --steps 20 --no-graph > gpurun_out/bench_c2.log 2>&1; echo c2=$?
cp bench_detail_n1.json gpurun_out/bench_detail_c2.json
for w in 2 4 8; do
  timeout 900 python bench.py --simulate-world $w --steps 20 >> gpurun_out/simulate_world.jsonl 2>> gpurun_out/simulate_world.err; echo sim$w=$?
done
timeout 900 python bench.py --maturity > gpurun_out/maturity.log 2>&1; echo mat=$?
