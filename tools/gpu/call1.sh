set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 tools/_build/peaks > gpurun_out/peaks.json 2> gpurun_out/peaks.err; echo peaks rc=$?
timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_ -s 10 -c 11 -o gpurun_out/c2k4_full python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_ncu.log 2>&1; echo ncu rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -3 gpurun_out/gputest.log
