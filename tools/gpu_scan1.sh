set -x
timeout 1200 python -m pytest tests/test_ivf_gpu.py tests/test_ivf_small_gpu.py tests/test_mature_gpu.py tests/test_graph_gpu.py tests/test_fp8_gpu.py tests/test_nccl_single_gpu.py tests/test_robustness_gpu.py -q -x > gpurun_out/scan1_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/scan1_tests.log
timeout 300 python tools/ivf_step_probe.py
timeout 300 python tools/ivf_step_probe.py --n 21015324
