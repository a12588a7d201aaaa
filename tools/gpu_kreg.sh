set -x
timeout 1200 python -m pytest tests/test_flat_gpu.py tests/test_fp8_gpu.py tests/test_sharded_gpu.py tests/test_robustness_gpu.py -x -q > gpurun_out/kreg_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/kreg_tests.log
for e in 0 4; do
 for n in 1000000:256 2626916:512 21015324:512; do
  SA_LIBRARY=tuning SA_EXPERIMENT=$e timeout 300 python tools/flat_probe.py --n ${n%%:*} --nq ${n##*:} --reps 10
 done
done
