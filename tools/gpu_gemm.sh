set -x
timeout 300 python tools/entry_probe.py; echo entry=$?
timeout 1200 python -m pytest tests/test_ivf_gpu.py tests/test_graph_gpu.py tests/test_mature_gpu.py tests/test_graph_mature_gpu.py tests/test_flat_gpu.py tests/test_sharded_gpu.py tests/test_sharded_comm_gpu.py -x -q > gpurun_out/gemm_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/gemm_tests.log
ncu --nvtx --nvtx-include "probe/" --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/entry_launches3.csv timeout 600 python tools/entry_probe.py > gpurun_out/entry_ncu3.log 2>&1
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 2>&1 | grep -o '"graph_search": [0-9.]*\|"ivf_probe": [0-9.]*\|"ms_per_batch": [0-9.]*\|"recall": [0-9.]*' | head -4
