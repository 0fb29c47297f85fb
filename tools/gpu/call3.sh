set -x
for v in "KCG_COMBINE=0" "KCG_COMBINE=1"; do
  echo "== $v"
  env $v timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 3 2>&1 | tail -1 | cut -c1-90
  env $v timeout 300 python tools/prof_count.py --config 3 --k 4 --reps 3 2>&1 | tail -1 | cut -c1-90
  env $v timeout 300 python tools/prof_count.py --config 2 --k 5 --reps 2 2>&1 | tail -1 | cut -c1-90
  env $v timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 2>&1 | tail -1 | cut -c1-90
  env $v timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1 | cut -c1-90
done
timeout 300 tests/cpp/bin/api_bench 2 5 0
timeout 600 tests/cpp/bin/api_bench 5 2 0
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
