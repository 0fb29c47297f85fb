timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fill_kernel|outdeg_kernel" --csv --log-file gpurun_out/c5_dag2.csv python tools/prof_c5.py 5 total > /dev/null 2>&1
grep -v "^==" gpurun_out/c5_dag2.csv | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>10 and r[0].isdigit(): print(r[0], r[4][:40], r[-1])
"
