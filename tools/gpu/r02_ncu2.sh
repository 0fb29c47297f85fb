set -x
timeout 300 python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_ -s 10 -c 10 -o gpurun_out/c2k4_full python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_ncu.log 2>&1; echo ncu rc=$?
timeout 600 python tools/prof_c5.py 5 total > gpurun_out/c5_plain.log 2>&1; echo c5 rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:count_ --csv --log-file gpurun_out/c5_launches.csv python tools/prof_c5.py 5 total > gpurun_out/c5_ncu.log 2>&1; echo ncu5 rc=$?
