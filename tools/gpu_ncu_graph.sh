set -x
timeout 1200 ncu --nvtx --nvtx-include "timed_graph/" --set full --import-source on --clock-control none -k regex:"graph_search|score_gemm|select_dense" -c 3 -o gpurun_out/prof_graph_step_r2 -f python bench.py --mode graph --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_graph_step.log 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_flat_gpu.py -q -x -k debug_scores > gpurun_out/dbg_scores.log 2>&1; echo dbg=$?; tail -2 gpurun_out/dbg_scores.log
