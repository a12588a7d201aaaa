set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
timeout 600 ./tools/gather_probe > gpurun_out/gather_probe.txt 2>&1
cat gpurun_out/gather_probe.txt
TOOLS="memcheck racecheck synccheck" CASE_TIMEOUT=400 timeout 3000 bash tools/run_sanitize.sh
