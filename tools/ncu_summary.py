import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
h=rows[0]
want=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__cycles_elapsed.avg','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_bytes.sum','smsp__average_warp_latency_issue_stalled_wait','launch__grid_size','launch__block_size']
for r in rows[2:]:
  for w in want:
    if w in h: print(w, rows[1][h.index(w)], r[h.index(w)])
