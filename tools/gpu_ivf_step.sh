set -x
timeout 300 python tools/ivf_step_probe.py
timeout 600 ncu --nvtx --nvtx-include "ivf_step/" --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ivf_step_launches.csv python tools/ivf_step_probe.py --reps 2 > gpurun_out/ivf_step_ncu.log 2>&1
