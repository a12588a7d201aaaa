set -x
python -m pytest tests -x -q -m gpu -s 2>&1 | grep -E "passed|failed|Error|error|assert|certified|parity:|touched|near-tie|uncertified" | tail -30
for e in "" "SA_EXPERIMENT=1" "SA_EXPERIMENT=3" "SA_SEED_ROWS=16384" "SA_SEED_ROWS=32768" "SA_SEED_ROWS=65536"; do
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 1000000 --nq 256
done
for e in "" "SA_EXPERIMENT=1" "SA_EXPERIMENT=3"; do
  env SA_LIBRARY=tuning $e python tools/flat_probe.py --n 1000000 --nq 256 --fp8 16
done
