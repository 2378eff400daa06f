#!/bin/bash
# usage: tools/ncu_summary.sh report.ncu-rep  -> key metrics + stall ratios + top opcodes/lines
rep=$1
ncu -i $rep --page raw --csv 2>/dev/null > /tmp/_raw.csv
ncu -i $rep --page source --csv --print-source=cuda,sass 2>/dev/null > /tmp/_src.csv
python3 - <<'PY'
import csv, re
r=list(csv.reader(open('/tmp/_raw.csv')))
h=r[0]; vals=r[2]; d=dict(zip(h,vals))
keys=['gpu__time_duration.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active',
'sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct','launch__registers_per_thread',
'smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','l1tex__t_bytes.sum',
'lts__t_sectors_srcunit_tex_op_read.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum','smsp__sass_thread_inst_executed_op_dmul_pred_on.sum','smsp__sass_thread_inst_executed_op_dadd_pred_on.sum','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','launch__shared_mem_per_block_dynamic']
for k in keys: print('%-64s %s'%(k, d.get(k)))
for k in h:
    if re.search(r'smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio',k):
        try:
            if float(d[k])>0.05: print('  stall %-30s %s'%(k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''), d[k]))
        except: pass
PY
python3 $(dirname $0)/ncu_source_summary.py /tmp/_src.csv 25 2>/dev/null
