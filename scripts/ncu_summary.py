import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines()))
h=r[0]; u=r[1]; v=r[2]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','dram__throughput.avg.pct_of_peak_sustained_elapsed','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','sm__cycles_elapsed.avg.per_second','launch__grid_size','launch__block_size']
for k in keys:
  if k in h: print(f'{k:60s} {v[h.index(k)]} {u[h.index(k)]}')
st=[(k,float(v[i])) for i,k in enumerate(h) if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued') and v[i].replace('.','').isdigit()]
st.sort(key=lambda x:-x[1]); tot=sum(x[1] for x in st)
print('stalls:', ', '.join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={100*x/tot:.0f}%" for k,x in st[:8]))
