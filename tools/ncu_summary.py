"""Summarise an ncu --page raw --csv export (one or more launches): duration, issue, pipes, stalls.
usage: python tools/ncu_summary.py raw.csv [launch_index]"""
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[0]; data=rows[2 + (int(sys.argv[2]) if len(sys.argv) > 2 else 0)]
def g(k):
    return data[hdr.index(k)] if k in hdr else None
for k in ['gpu__time_duration.sum','smsp__inst_executed.sum','thread_inst_executed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__thread_inst_executed_per_inst_executed.ratio','launch__registers_per_thread','dram__bytes_read.sum','dram__bytes_write.sum','launch__grid_size','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active']:
    print(k, g(k))
st=[(h,data[i]) for i,h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued') and data[i] not in ('0','')]
tot=sum(float(v) for _,v in st)
for h,v in sorted(st,key=lambda t:-float(t[1])): print('  %-60s %5.1f%%'%(h.replace('smsp__pcsamp_warps_issue_stalled_',''),100*float(v)/tot))
