set -x
SA_LIBRARY=tuning timeout 900 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 --pf 0,4,8,12,0 > gpurun_out/graph_hint.json 2> gpurun_out/graph_hint.log
grep -o '"pf": "[0-9]*"\|"graph_search": [0-9.]*' gpurun_out/graph_hint.log
timeout 900 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 2>&1 | grep -o '"graph_search": [0-9.]*' | head -1
