import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines())); h=r[0]; v=r[2]
d=dict(zip(h,v))
keys=['gpu__time_duration.sum','sm__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_shared_mem','sm__warps_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum']
for k in keys:
    for kk in d:
        if kk==k or kk.endswith('.'+k): print(k, d[kk]); break
    else: print(k,'?')
for a,c in d.items():
    if 'smsp__average_warps_issue_stalled' in a and a.endswith('_per_issue_active.ratio'):
        try:
            if float(c)>0.1: print('  stall',a.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''),c)
        except: pass
