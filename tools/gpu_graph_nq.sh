set -x
for nq in 512 1024 2048; do
timeout 600 python tools/graph_probe.py --degree 48 --widths 4 --entries 16 --ranges 100 --nq $nq 2>&1 | tail -2
done
