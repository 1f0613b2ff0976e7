"""Per-CUDA-source-line aggregation of an ncu --set full report's source page
(`--print-source cuda,sass`, compiled with -lineinfo): warp-level
instructions executed and stall samples per line, per kernel.

  python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kre], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(txt))
hdr = None
fpath = fn = None
line = None
agg = {}
kern_tot = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None:
        continue
    if r[0]:   # a CUDA source line (its SASS rows follow)
        line = (fpath, int(r[0]), r[1].strip()[:90])
        continue
    # SASS row of the current source line
    try:
        n = float(r[ix] or 0)
        s = float(r[isamp] or 0)
    except (ValueError, IndexError):
        continue
    key = (fn, line)
    a = agg.setdefault(key, [0.0, 0.0, 0])
    a[0] += n
    a[1] += s
    a[2] += 1
    t = kern_tot.setdefault(fn, [0.0, 0.0])
    t[0] += n
    t[1] += s
for fn, (ti, ts) in kern_tot.items():
    print("== %s  instr %.3g  samples %.0f" % (fn[:80], ti, ts))
    items = [(v, k[1]) for k, v in agg.items() if k[0] == fn]
    byfile = {}
    for v, ln in items:
        byfile[ln[0]] = byfile.get(ln[0], 0) + v[0]
    print("   instr by file: " + ", ".join("%s %.1f%%" % (f, 100 * x / max(ti, 1)) for f, x in sorted(byfile.items(), key=lambda z: -z[1])))
    print("   %6s %6s %4s  line" % ("instr%", "stall%", "sass"))
    for v, ln in sorted(items, key=lambda z: -z[0][0])[:top]:
        print("   %6.2f %6.2f %4d  %s:%d  %s" % (100 * v[0] / max(ti, 1), 100 * v[1] / max(ts, 1), v[2], ln[0], ln[1], ln[2]))
