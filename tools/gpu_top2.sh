set -x
timeout 1500 python -m pytest tests/test_graph_gpu.py tests/test_graph_mature_gpu.py tests/test_retriever_gpu.py tests/test_select_ties_gpu.py tests/test_flat_gpu.py -q -x > gpurun_out/top2_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/top2_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 900 ncu --nvtx --nvtx-include "timed_graph/" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_graph_top2.csv python bench.py --mode graph --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_top2.log 2>&1; echo launches=$?
timeout 900 python bench.py --mode graph --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_graph_top2.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_graph_top2.log | cut -c1-300
