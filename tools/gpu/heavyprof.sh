SKIP=1 TOP=70 tools/ncu_sum.sh c5_heavy2 count_heavy4 -- python tools/prof_c5.py 5 total
