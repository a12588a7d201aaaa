set -x
timeout 1500 python -m pytest tests/test_graph_gpu.py tests/test_graph_mature_gpu.py tests/test_retriever_gpu.py tests/test_fullsize_gpu.py -q -x > gpurun_out/inplace_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/inplace_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 2>&1 | grep -o '"graph_search": [0-9.]*\|"ivf_probe": [0-9.]*\|"stage": [0-9.]*\|"ms_per_batch": [0-9.]*\|"recall": [0-9.]*' | head -5
