timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_|fill_|outdeg|Scan|Reduce" --csv --log-file gpurun_out/c5_dag.csv python tools/prof_c5.py 5 total > /dev/null 2>&1
python3 - <<'P'
import csv
hdr=None
for r in csv.reader(open('gpurun_out/c5_dag.csv')):
    if hdr is None:
        if r and r[0]=='ID': hdr=r
        continue
    d=dict(zip(hdr,r))
    ms=float(d['Metric Value'].replace(',',''))/1e6
    if ms>0.05: print(d['ID'], d['Kernel Name'][:60], d['Grid Size'], '%.3f ms'%ms)
P
