set -x
SA_LIBRARY=tuning timeout 600 python tools/graph_phase_probe.py --L 64,100,160 > gpurun_out/graph_phase.log 2>&1
cat gpurun_out/graph_phase.log | tail -5
