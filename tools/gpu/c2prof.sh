SKIP=0 TOP=45 tools/ncu_sum.sh c2k4_cta_big count_cta -- python tools/prof_count.py --config 2 --k 4 --reps 1
