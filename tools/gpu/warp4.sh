tools/ncu_sum.sh c3k4_warp_b count_warp -- python tools/prof_count.py --config 3 --k 4 --reps 1
