set -x
for bd in 0 16 1000000; do
 for n in 1000000:256 2626916:512 21015324:512; do
  COUNT=1 SA_LIBRARY=tuning SA_BOUND_DENSE=$bd timeout 300 python tools/flat_probe.py --n ${n%%:*} --nq ${n##*:} --reps 10
 done
done
