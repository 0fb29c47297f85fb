# quick A/B: counting times on the main configs + the parity tests
set -x
for c in "2 4" "3 4" "2 5" "4 6"; do set -- $c; timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 2>&1 | tail -1 | cut -c1-120; done
timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1 | cut -c1-120
timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 2 --pv 2>&1 | tail -1 | cut -c1-120
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shard.py -x -q 2>&1 | tail -3
