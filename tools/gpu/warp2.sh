timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c3k4_warp python tools/prof_count.py --config 3 --k 4 --reps 1 > gpurun_out/c3k4_warp.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c4k6_warp python tools/prof_count.py --config 4 --k 6 --reps 1 > gpurun_out/c4k6_warp.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c4k6pv_warp python tools/prof_count.py --config 4 --k 6 --reps 1 --pv > gpurun_out/c4k6pv_warp.log 2>&1; echo rc=$?
ls -la gpurun_out
