set -x
ncu --set full --import-source on --clock-control none -k regex:flat_scan_topk -s 3 -c 1 -o gpurun_out/prof_c2_flat -f timeout 600 python tools/flat_probe.py --n 1000000 --nq 256 --reps 2 > gpurun_out/ncu_c2.log 2>&1
tail -3 gpurun_out/ncu_c2.log
