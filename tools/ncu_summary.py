"""Per-kernel summary of an ncu --set full report: duration, registers,
occupancy, issue activity, top stall reasons and busiest pipes."""
import csv, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(txt))
hdr = rows[0]
def f(r, k):
    try:
        return float(r[hdr.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return float("nan")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print("== %s  grid %s block %s" % (name[:60], r[hdr.index("Grid Size")], r[hdr.index("Block Size")]))
    print("   %.3f ms  regs %d  warps/sched active %.2f eligible %.2f  issue-active %.1f%%  ipc %.2f" % (
        f(r, "gpu__time_duration.sum") / 1e6, f(r, "launch__registers_per_thread"),
        f(r, "smsp__warps_active.avg.per_cycle_active"), f(r, "smsp__warps_eligible.avg.per_cycle_active"),
        f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"), f(r, "sm__inst_executed.avg.per_cycle_active")))
    st = [(f(r, h), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
          for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    st = sorted([x for x in st if x[0] == x[0]], reverse=True)[:7]
    print("   stalls: " + ", ".join("%s %.2f" % (n, v) for v, n in st))
    pp = [(f(r, h), h.replace("sm__inst_executed_pipe_", "").replace(".avg.pct_of_peak_sustained_active", ""))
          for h in hdr if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active")]
    pp = sorted([x for x in pp if x[0] == x[0]], reverse=True)[:5]
    print("   pipes: " + ", ".join("%s %.1f%%" % (n, v) for v, n in pp))
    print("   dram %.1f MB  l1 hit %.1f%%  l2 hit %.1f%%" % (
        (f(r, "dram__bytes_read.sum") + f(r, "dram__bytes_write.sum")) / 1e6,
        f(r, "l1tex__t_sector_hit_rate.pct"), f(r, "lts__t_sector_hit_rate.pct")))
