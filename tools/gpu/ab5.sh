for v in paper_2002_10047_b200/lib/libkcg.so tools/_build/libkcg_*.so; do
  echo "== $v"
  for c in "2 4" "3 4" "3 5"; do set -- $c; KCG_LIB=$PWD/$v timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 2>&1 | tail -1 | cut -c1-80; done
done
