timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_hubs.py tests/test_gpu_peel.py -x -q -m gpu 2>&1 | tail -2
for c in "2 4" "3 4" "1 4"; do set -- $c; timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 --pv 2>&1 | tail -1 | cut -c1-80; done
timeout 900 python tools/prof_c5.py 5 pv 2>&1 | tail -1 | cut -c1-80
