set -x
python -m pytest tests/test_sharded_comm_gpu.py tests/test_accounting_gpu.py -x -q 2>&1 | tail -30
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/condgraph_probe tools/condgraph_probe.cu
/usr/local/cuda/bin/compute-sanitizer --tool synccheck /tmp/condgraph_probe direct 2>&1 | tail -4
/usr/local/cuda/bin/compute-sanitizer --tool synccheck /tmp/condgraph_probe graph 2>&1 | tail -8
TOOLS="racecheck synccheck" CASES="merge graph mature" CASE_TIMEOUT=300 tools/run_sanitize.sh
python -m pytest tests -x -q -m gpu 2>&1 | tail -15
