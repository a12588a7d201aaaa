set -x
for r in 0 8192 16384 32768 65536; do SA_LIBRARY=tuning SA_SEED_ROWS=$r timeout 300 python tools/flat_probe.py --n 1000000 --nq 256; done
for r in 0 16384 65536; do SA_LIBRARY=tuning SA_SEED_ROWS=$r timeout 300 python tools/flat_probe.py --n 2626916 --nq 512; done
