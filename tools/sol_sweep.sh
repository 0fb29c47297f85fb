#!/bin/bash
# Speed-of-light sweep of the counting launches for every (config, k):
# per-launch duration, SM throughput (% of peak issue), DRAM and L2 bytes.
# Usage (on the GPU box): bash tools/sol_sweep.sh OUTDIR
out=${1:-gpurun_out/sol}
mkdir -p "$out"
M=gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed.sum
for ck in "1 3" "1 4" "2 4" "2 5" "3 4" "3 5" "3 6" "3 7" "3 8" "4 6" "4 8"; do
  set -- $ck
  ncu --metrics $M --clock-control none --csv -k regex:count_ --log-file "$out/c$1k$2.csv" \
      python tools/prof_count.py --config $1 --k $2 --reps 1 > /dev/null 2>&1
  echo "c$1 k$2 rc=$?"
done
ncu --metrics $M --clock-control none --csv -k regex:count_ --log-file "$out/c4k6pv.csv" \
    python tools/prof_count.py --config 4 --k 6 --reps 1 --pv > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv -k regex:count_ --log-file "$out/c5k4.csv" \
    python tools/prof_c5.py 5 total > /dev/null 2>&1
echo done
