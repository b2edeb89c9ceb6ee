#!/bin/bash
# Summarise an ncu report (details, stall mix, DRAM bytes, hot source lines) as text.
#   tools/ncu_summary.sh gpurun_out/x.ncu-rep [launch-skip] > profiles/x.txt
rep=$1; skip=${2:-0}
echo "# ncu summary of $rep (launch-skip $skip)"
ncu -i "$rep" --page details --launch-skip "$skip" --launch-count 1 2>/dev/null | grep -E "^  [a-zA-Z_]|Grid Size|Block Size|Duration|DRAM Throughput|Memory Throughput|Registers Per|Achieved Occupancy|Theoretical Occupancy|L2 Hit|L1/TEX Hit|Executed Ipc A|Issue Slots Busy|Dynamic Shared|Achieved Active|Compute \(SM\)"
echo "## raw"
ncu -i "$rep" --page raw --csv --launch-skip "$skip" --launch-count 1 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); hdr,units,vals=rows[0],rows[1],rows[2]
out=[]
for h,u,v in zip(hdr,units,vals):
    if h in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','smsp__inst_executed.sum','lts__t_sectors_srcunit_tex_op_read.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread'): print(h,u,v)
    if 'pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued'):
        try: out.append((float(v.replace(',','')),h))
        except: pass
t=sum(v for v,h in out) or 1
print('## stall mix (pc sampling)')
for v,h in sorted(out,reverse=True)[:8]: print(f'{v/t:6.1%}',h.replace('smsp__pcsamp_warps_issue_stalled_',''))
"
echo "## hot source lines"
ncu -i "$rep" --page source --csv --print-source cuda,sass --launch-skip "$skip" --launch-count 1 2>/dev/null > /tmp/_ncu_src.csv
python3 "$(dirname "$0")/line_hot.py" /tmp/_ncu_src.csv 20
