# graph search: L2-prefetch modes (SA_GRAPH_PF, tuning library) at the bench setting
set -x
SA_LIBRARY=tuning timeout 900 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 --pf 0,1,2,3 > gpurun_out/graph_pf.json 2> gpurun_out/graph_pf.log
tail -5 gpurun_out/graph_pf.log
