set -x
for nb in 0 1; do
 for n in 1000000:256 2626916:512 21015324:512; do
  SA_LIBRARY=tuning SA_NO_BOUND=$nb timeout 300 python tools/flat_probe.py --n ${n%%:*} --nq ${n##*:} --reps 10
 done
done
SA_LIBRARY=tuning SA_NO_BOUND=1 SA_EXPERIMENT=3 timeout 300 python tools/flat_probe.py --n 1000000 --nq 256
