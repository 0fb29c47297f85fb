# A/B of counting-kernel variants (env knobs) on configs 2/3/4/5
set -x
for v in "KCG_LEAN_PAD=0 KCG_COMBINE=0" "KCG_LEAN_PAD=1 KCG_COMBINE=0" "KCG_LEAN_PAD=0 KCG_COMBINE=1" "KCG_LEAN_PAD=1 KCG_COMBINE=1"; do
  echo "== $v"
  env $v timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 3 2>&1 | tail -1
  env $v timeout 300 python tools/prof_count.py --config 3 --k 4 --reps 3 2>&1 | tail -1
done
for v in "KCG_COMBINE=0" "KCG_COMBINE=1"; do
  echo "== $v"
  env $v timeout 300 python tools/prof_count.py --config 2 --k 5 --reps 2 2>&1 | tail -1
  env $v timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 2>&1 | tail -1
  env $v timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1
done
