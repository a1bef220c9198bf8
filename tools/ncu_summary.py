import csv, subprocess, sys
def summ(rep):
    out = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rows=list(csv.reader(out.splitlines()))
    h=rows[0]; u=rows[1]; v=rows[2]
    want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','l1tex__t_sector_hit_rate.pct','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum','launch__shared_mem_per_block_dynamic','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem']
    res={}
    for i,name in enumerate(h):
        if name in want: res[name]=(v[i],u[i])
    items=[]
    for i,name in enumerate(h):
        if 'smsp__pcsamp_warps_issue_stalled' in name and not name.endswith('not_issued'):
            try: items.append((float(v[i]), name.replace('smsp__pcsamp_warps_issue_stalled_','')))
            except: pass
    items.sort(reverse=True); tot=sum(x for x,_ in items) or 1
    return res, [(n, round(100*x/tot,1)) for x,n in items[:8]]
if __name__=='__main__':
    for rep in sys.argv[1:]:
        res, st = summ(rep)
        print('==', rep)
        for k,(val,un) in res.items(): print(f'  {k}: {val} {un}')
        print('  stalls:', st)
