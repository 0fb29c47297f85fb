for c in "3 6" "3 7" "3 8" "2 5" "4 8"; do set -- $c; timeout 600 python tools/prof_count.py --config $1 --k $2 --reps 2 2>&1 | tail -1 | cut -c1-80; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -2
