set -x
for c in "2 4" "3 4" "2 5" "4 6" "4 8"; do set -- $c; timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 2>&1 | tail -1 | cut -c1-100; done
timeout 300 python tools/prof_count.py --config 4 --k 6 --reps 2 --pv 2>&1 | tail -1 | cut -c1-100
KCG_COMBINE=1 timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 3 2>&1 | tail -1 | cut -c1-100
KCG_COMBINE=0 timeout 300 python tools/prof_count.py --config 3 --k 4 --reps 3 2>&1 | tail -1 | cut -c1-100
timeout 300 tests/cpp/bin/api_bench 2 5 0
timeout 900 tests/cpp/bin/api_bench 5 2 0
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_ -s 10 -c 11 -o gpurun_out/c2k4_swz python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_ncu4.log 2>&1; echo ncu rc=$?
