#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py; logs in gpurun_out/sanitize_<tool>.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CASES="${CASES:-flat1 flat2 flatk merge ivf ivfsmall mature graph graph_mature fp8 host}"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool" > gpurun_out/sanitize_$tool.txt
  for c in $CASES; do
    echo "-- case $c" >> gpurun_out/sanitize_$tool.txt
    timeout ${CASE_TIMEOUT:-600} /usr/local/cuda/bin/compute-sanitizer --tool $tool \
      --print-limit 20 python tools/sanitize_cases.py $c >> gpurun_out/sanitize_$tool.txt 2>&1
    echo "-- case $c rc=$?" >> gpurun_out/sanitize_$tool.txt
  done
done
grep -h "rc=\|ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize cases" gpurun_out/sanitize_*.txt
