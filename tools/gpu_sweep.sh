set -x
timeout 1800 python bench.py --sweep > gpurun_out/sweep.log 2>&1; echo sweep=$?
tail -c 600 gpurun_out/sweep.log
