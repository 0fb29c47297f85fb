set -x
timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_ -s 10 -c 11 -o gpurun_out/c2k4_full python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_ncu.log 2>&1; echo ncu rc=$?
timeout 300 python tools/prof_direct.py 5 2 > gpurun_out/c5dir_plain.log 2>&1; echo dplain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/c5dir_launches.csv python tools/prof_direct.py 5 2 > gpurun_out/c5dir_ncu.log 2>&1; echo ncu rc=$?
