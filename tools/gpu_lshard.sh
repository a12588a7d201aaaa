set -x
timeout 1200 python -m pytest tests/test_list_shard_gpu.py tests/test_sharded_comm_gpu.py tests/test_nccl_single_gpu.py tests/test_ivf_gpu.py tests/test_ivf_small_gpu.py -q -x > gpurun_out/lshard_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/lshard_tests.log
