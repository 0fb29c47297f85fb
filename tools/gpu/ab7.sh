for v in paper_2002_10047_b200/lib/libkcg.so tools/_build/libkcg_*.so; do
  echo "== $v"
  for c in "4 6" "4 8" "3 6" "2 5"; do set -- $c; KCG_LIB=$PWD/$v timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 2 2>&1 | tail -1 | cut -c1-80; done
  KCG_LIB=$PWD/$v timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1 | cut -c1-80
done
