set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo gputest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
cp bench_detail_n1.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/gputest.log
