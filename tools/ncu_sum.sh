#!/bin/bash
# On the GPU box: one `ncu --set full` capture of the first launch matching
# KERNEL_REGEX, reduced to text (key raw metrics + per-source-line totals) so
# the result fits gpurun_out/.   usage: ncu_sum.sh NAME KERNEL_REGEX -- command...
name=$1; re=$2; shift 3
rep=/tmp/$name.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s ${SKIP:-0} -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1 || { echo "ncu failed"; tail -5 gpurun_out/$name.log; exit 1; }
{
  ncu -i $rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for row in r[2:]:
    for i,x in enumerate(h):
        if '__' in x or x=='Kernel Name': print(x, '=', row[i])
"
  ncu -i $rep --page details --csv 2>/dev/null | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>14 and ('Stall' in r[12] or 'stall' in r[12].lower()): print(r[12], r[14])
" | head -0
  python3 tools/ncu_lines.py $rep ::regex:$re:1 ${TOP:-60}
} > gpurun_out/$name.txt 2>&1
rm -f $rep
