set -x
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 2>&1 | grep -o '"graph_search": [0-9.]*\|"recall": [0-9.]*' | head -2
timeout 600 python tools/entry_probe.py
