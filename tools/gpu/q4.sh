timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -3
for c in "2 5" "3 5" "3 6" "3 8" "4 6" "4 8"; do set -- $c; timeout 600 python tools/prof_count.py --config $1 --k $2 --reps 2 2>&1 | tail -1 | cut -c1-90; done
timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1 | cut -c1-90
