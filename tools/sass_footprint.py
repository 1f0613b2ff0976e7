"""Per-section SASS footprint from an ncu report (source page, sass view):
static instruction count, executed warp-instructions, stall samples and
instruction-fetch (no_inst) stall samples, plus the hottest 4 KB windows."""
import csv, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
secs, cur, hdr = [], None, None
for r in csv.reader(txt):
    if not r:
        continue
    if r[0] == "Address":
        hdr = r
        cur = []
        secs.append(cur)
        continue
    if r[0].startswith("0x") and cur is not None:
        g = lambda k: float(r[hdr.index(k)]) if r[hdr.index(k)] not in ("", "-") else 0.0
        cur.append((int(r[0], 16), r[1].strip(), g("Instructions Executed"), g("Warp Stall Sampling (All Samples)"),
                    g("stall_no_inst"), g("stall_barrier")))
for i, s in enumerate(secs):
    if not s:
        continue
    n = len(s)
    ex = sum(x[2] for x in s)
    smp = sum(x[3] for x in s)
    ni = sum(x[4] for x in s)
    live = sum(1 for x in s if x[2] > 0)
    print("section %d: %d instr (%.0f KB), %d executed at least once, %.3g warp-instr, samples %d, no_inst %d (%.1f%%)"
          % (i, n, n * 16 / 1024, live, ex, smp, ni, 100 * ni / max(smp, 1)))
    base = s[0][0]
    win = {}
    for a, src, e, sm, nn, b in s:
        w = (a - base) // 4096
        t = win.setdefault(w, [0, 0, 0, 0])
        t[0] += e; t[1] += sm; t[2] += nn; t[3] += 1 if e > 0 else 0
    top = sorted(win.items(), key=lambda kv: -kv[1][1])[:12]
    for w, (e, sm, nn, lv) in sorted(top):
        print("   +%4d KB  exec %.3g  samples %6d  no_inst %5d  live %d" % (w * 4, e, sm, nn, lv))
