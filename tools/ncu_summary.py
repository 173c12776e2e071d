"""Compact summary of a one-kernel `ncu --set full` report: launch shape,
duration, FP64-pipe and SM utilisation, DRAM traffic, occupancy, and the
source lines with the most warp-stall samples.
usage: ncu_summary.py REP [N_LINES]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
def g(name):
    v = m.get(name)
    return "%s %s" % v if v else "n/a"
keys = [
    ("kernel", "Kernel Name"), ("grid", "launch__grid_size"),
    ("block", "launch__block_size"), ("registers/thread", "launch__registers_per_thread"),
    ("duration", "gpu__time_duration.sum"),
    ("SM clock", "smsp__cycles_elapsed.avg.per_second"),
    ("FP64 pipe (inst executed, % of peak, active)", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe cycles active (% elapsed)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput (% elapsed)", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue active (% active)", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("DRAM read", "dram__bytes_read.sum"), ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput (% elapsed)", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
    ("achieved occupancy", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("DADD thread-instructions", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"),
    ("DMUL thread-instructions", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"),
    ("DFMA thread-instructions", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"),
]
for label, key in keys:
    print("%-48s %s" % (label, g(key)))
print()
print("top source lines by warp-stall samples:")
out = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "ncu_lines.py"),
                      rep, ".", str(nl)], capture_output=True, text=True).stdout
print(out)
