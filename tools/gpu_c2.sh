set -x
timeout 900 python bench.py --config c2 --steps 20 --no-graph > gpurun_out/bench_c2.log 2>&1; echo c2=$?
cp gpurun_out/bench_detail_n1.json gpurun_out/bench_detail_c2.json
tail -1 gpurun_out/bench_c2.log | cut -c1-400
