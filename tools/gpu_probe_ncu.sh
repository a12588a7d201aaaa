set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_scan|select_dense|merge" -c 40 --csv --log-file gpurun_out/entry_launches.csv timeout 600 python tools/entry_probe.py > gpurun_out/entry_ncu.log 2>&1
SA_LIBRARY=tuning SA_EXPERIMENT=1 timeout 600 python tools/entry_probe.py
