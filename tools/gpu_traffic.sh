# one ncu --set full capture each of the IVF list scan and the exact flat scan at the bench
# configuration (C3, batch 512, top-10; IVF nprobe 48): DRAM traffic for bench.py's roofline.
# The exact step launches the seed sub-scan first (one flat_scan_topk launch), hence -s 1.
set -x
timeout 1200 ncu --nvtx --nvtx-include "timed_ivf/" --set full --import-source on --clock-control none -k regex:ivf_scan -c 1 -o gpurun_out/prof_ivf_r2 -f python bench.py --mode ivf --nprobe 48 --steps 2 --warmup 3 --no-cpu-baseline --no-graph --no-fp8 > gpurun_out/ncu_ivf.log 2>&1; echo ivf=$?
timeout 1200 ncu --nvtx --nvtx-include "timed_exact/" --set full --import-source on --clock-control none -k regex:flat_scan_topk -s 1 -c 1 -o gpurun_out/prof_exact_r2 -f python bench.py --mode exact --steps 2 --warmup 3 --no-cpu-baseline --no-graph --no-fp8 > gpurun_out/ncu_exact.log 2>&1; echo exact=$?
