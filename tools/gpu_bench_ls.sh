set -x
SA_BENCH_LIST_SHARD=1 timeout 900 python bench.py --mode ivf --nprobe 48 --steps 10 --no-cpu-baseline --no-graph > gpurun_out/bench_ls.log 2>&1; echo ls=$?
tail -1 gpurun_out/bench_ls.log | cut -c1-600
timeout 900 python bench.py --simulate-world 8 --steps 20 > gpurun_out/sim8.log 2>&1; echo sim=$?
tail -1 gpurun_out/sim8.log
