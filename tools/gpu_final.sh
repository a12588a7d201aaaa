# full GPU pass: smoke, GPU tests, default bench, the graph step's launch list, one ncu --set full
# of the headline kernel and one of the probe GEMM
set -x
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo gputest=$?
tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
cp gpurun_out/bench_detail_n1.json gpurun_out/bench_detail_default.json   # before the ncu runs overwrite it
tail -1 gpurun_out/bench.log | cut -c1-400
timeout 900 ncu --nvtx --nvtx-include "timed_graph/" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_graph.csv python bench.py --mode graph --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"graph_search|score_gemm" -s 6 -c 2 -o gpurun_out/prof_graph_r2 -f python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 > gpurun_out/ncu_full.log 2>&1; echo full=$?
