set -x
for c in "2 4" "3 4" "4 6"; do set -- $c; timeout 300 python tools/prof_count.py --config $1 --k $2 --reps 3 2>&1 | tail -1 | cut -c1-100; done
timeout 300 tests/cpp/bin/api_bench 2 5 0
KCG_REGISTER=0 timeout 300 tests/cpp/bin/api_bench 2 5 0
timeout 900 tests/cpp/bin/api_bench 5 2 0
timeout 900 tests/cpp/bin/api_bench 5 1 1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/prof_direct.py 5 2 > gpurun_out/c5dir_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5dir_launches.csv python tools/prof_direct.py 5 2 > gpurun_out/c5dir_ncu.log 2>&1; echo ncu rc=$?
