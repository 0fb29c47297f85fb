set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "hub1500 or rmat12 or planted" 2>&1 | tail -5
timeout 600 python tools/prof_c5.py 5 total 2>&1 | tail -2
KCG_TILED=0 timeout 600 python tools/prof_c5.py 5 total 2>&1 | tail -2
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:count_heavy --csv --log-file gpurun_out/c5_heavy_launches.csv python tools/prof_c5.py 5 total > gpurun_out/c5_ncu.log 2>&1; echo ncu5 rc=$?
