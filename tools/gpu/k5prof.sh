timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:count_ --csv --log-file gpurun_out/c2k5_launches.csv python tools/prof_count.py --config 2 --k 5 --reps 1 > /dev/null 2>&1
grep -v "^==" gpurun_out/c2k5_launches.csv | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>10 and r[0].isdigit(): print(r[0], r[4][:70], r[-1])
"
SKIP=2 TOP=70 tools/ncu_sum.sh c2k5_cta count_cta -- python tools/prof_count.py --config 2 --k 5 --reps 1
