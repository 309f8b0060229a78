"""Summarise one ncu --set full capture: key counters + top source lines by warp-stall samples.
python tools/ncu_report.py rep.ncu-rep "header comment" > profiles/ncu_<kernel>_<round>.txt"""
import csv, subprocess, sys
rep = sys.argv[1]
hdr = sys.argv[2] if len(sys.argv) > 2 else ""
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
     "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
     "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_issue_stalled_barrier.ratio",
     "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
print(f"# {hdr}")
print(f"# kernel: {v[h.index('Kernel Name')]}")
for m in M:
    if m in h:
        i = h.index(m)
        print(f"{m} = {v[i]} {u[i]}")
print("\n# warp-stall samples by source line (top 15)")
sys.stdout.flush()
subprocess.run([sys.executable, __file__.replace("ncu_report.py", "ncu_lines.py"), rep, "15"])
