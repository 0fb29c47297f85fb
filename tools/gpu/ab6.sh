timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -2
for v in paper_2002_10047_b200/lib/libkcg.so tools/_build/libkcg_*.so; do
  echo "== $v"
  for c in "2 4" "3 4"; do set -- $c; KCG_LIB=$PWD/$v timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 2>&1 | tail -1 | cut -c1-80; done
  KCG_LIB=$PWD/$v timeout 600 python tools/prof_c5.py 5 total 2>&1 | tail -1 | cut -c1-80
done
