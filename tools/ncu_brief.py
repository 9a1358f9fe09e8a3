"""Headline metrics + top stall reasons of one ncu report.  usage: python tools/ncu_brief.py rep.ncu-rep"""
import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines())); h=r[0]; v=r[-1]
keys=['gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.per_cycle_active','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','launch__occupancy_limit_shared_mem','launch__occupancy_limit_warps','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','lts__t_sectors_srcunit_tex_op_write.sum','l1tex__t_requests_pipe_lsu_mem_global_op_st.sum']
for i,n in enumerate(h):
    if n in keys: print(f'{n:70s} {v[i]}')
st=[(float(v[i].replace(',','') or 0),n) for i,n in enumerate(h) if n.startswith('smsp__average_warp_latency_issue_stalled') or (n.startswith('smsp__warp_issue_stalled') and n.endswith('per_warp_active.pct'))]
for x,n in sorted(st,reverse=True)[:8]: print(f'{n:70s} {x}')
