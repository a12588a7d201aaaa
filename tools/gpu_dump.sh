set -x
ncu --nvtx --nvtx-include "probe/" --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/entry_launches2.csv timeout 600 python tools/entry_probe.py > gpurun_out/entry_ncu2.log 2>&1
timeout 600 python tools/entry_probe.py
