# graph search rework: parity tests, then phase timings and q/s on the C3 graph
set -x
timeout 900 python -m pytest tests/test_graph_gpu.py tests/test_graph_mature_gpu.py tests/test_retriever_gpu.py -x -q > gpurun_out/graph_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/graph_tests.log
SA_LIBRARY=tuning timeout 600 python tools/graph_phase_probe.py --L 64,100,160 > gpurun_out/graph_phase2.log 2>&1
tail -3 gpurun_out/graph_phase2.log
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100,160 --fp8 0,1 > gpurun_out/graph_probe2.json 2> gpurun_out/graph_probe2.log
tail -4 gpurun_out/graph_probe2.log
