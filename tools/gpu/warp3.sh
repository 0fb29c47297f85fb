tools/ncu_sum.sh c3k4_warp count_warp -- python tools/prof_count.py --config 3 --k 4 --reps 1
tools/ncu_sum.sh c4k6_warp count_warp -- python tools/prof_count.py --config 4 --k 6 --reps 1
tools/ncu_sum.sh c4k6pv_warp count_warp -- python tools/prof_count.py --config 4 --k 6 --reps 1 --pv
