set -x
ncu --nvtx --nvtx-include "probe/" --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/entry_launches.csv timeout 600 python tools/entry_probe.py > gpurun_out/entry_ncu.log 2>&1
tail -3 gpurun_out/entry_ncu.log
SA_LIBRARY=tuning SA_EXPERIMENT=1 timeout 600 python tools/entry_probe.py
for e in 0 1 2 3; do SA_LIBRARY=tuning SA_EXPERIMENT=$e timeout 300 python tools/flat_probe.py --n 1000000 --nq 256; done
