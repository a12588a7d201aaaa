set -x
python -m pytest tests/test_flat_gpu.py tests/test_fp8_gpu.py -x -q 2>&1 | tail -3
for e in "" "SA_NO_SEED=1"; do
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 1000000 --nq 256
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 1000000 --nq 256 --fp8 16
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 21015324 --nq 512 --reps 10
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 21015324 --nq 512 --reps 10 --fp8 16
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 2626916 --nq 512 --reps 20
done
ncu --nvtx --nvtx-include "agent/" --metrics gpu__time_duration.sum --csv --log-file gpurun_out/agent_b1_launches.csv python tools/agent_step_probe.py 1 48
python tools/agent_step_probe.py 1 48; python tools/agent_step_probe.py 8 48
