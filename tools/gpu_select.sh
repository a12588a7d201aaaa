set -x
timeout 1200 python -m pytest tests/test_ivf_gpu.py tests/test_graph_gpu.py tests/test_mature_gpu.py tests/test_graph_mature_gpu.py tests/test_robustness_gpu.py tests/test_sharded_gpu.py -x -q > gpurun_out/select_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/select_tests.log
timeout 600 python tools/entry_probe.py
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 2>&1 | grep -o '"graph_search": [0-9.]*\|"ivf_probe": [0-9.]*\|"ms_per_batch": [0-9.]*' | head -3
