set -x
timeout 900 python -m pytest tests/test_nccl_single_gpu.py tests/test_sharded_comm_gpu.py tests/test_sharded_gpu.py tests/test_ivf_gpu.py -q -x > gpurun_out/nccl1_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/nccl1_tests.log
timeout 300 python tools/ivf_step_probe.py
