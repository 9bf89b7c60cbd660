"""Summarise an ncu --set full report: time, DRAM bytes, throughput percentages and the top
warp-stall reasons per kernel.   python scripts/ncu_summary.py gpurun_out/<report>.ncu-rep
"""
import csv, sys, collections, subprocess
rep = sys.argv[1]
raw = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines()))
h=r[0]; units=r[1]
keys=['gpu__time_duration.sum','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','l1tex__data_pipe_tc_wavefronts_mem_shared.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','lts__t_sectors_srcunit_tex_op_read.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','smsp__warps_active.avg.per_cycle_active','launch__registers_per_thread','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']
for row in r[2:]:
  print('=====', row[h.index('Kernel Name')][:70])
  for k in keys:
    if k in h: print('  %-70s %s %s'%(k, row[h.index(k)], units[h.index(k)]))
  items=[]
  for i,k in enumerate(h):
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
      try: items.append((float(row[i].replace(',','')),k))
      except: pass
  tot=sum(v for v,_ in items) or 1
  for v,k in sorted(items,reverse=True)[:8]: print('   %6.1f%% %s'%(100*v/tot,k.replace('smsp__pcsamp_warps_issue_stalled_','')))
