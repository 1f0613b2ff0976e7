"""Aggregate ncu 'cuda,sass' source-page samples per CUDA source line."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(txt))
agg = {}
fn = fp = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fp = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        fn = r[1][:45]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] and r[0] != "" and hdr:
        try:
            ln = int(r[0])
        except ValueError:
            continue
        s = float(r[4]) if r[4] not in ("", "-") else 0.0
        key = (fn, fp, ln)
        agg[key] = (agg.get(key, (0, ""))[0] + s, r[1][:100])
byk = {}
for (fn, fp, ln), (s, src) in agg.items():
    byk.setdefault(fn, []).append((s, fp, ln, src))
for fn, v in byk.items():
    tot = sum(x[0] for x in v) or 1
    print("==", fn, int(tot))
    byf = {}
    for s, fp, ln, src in v:
        byf[fp] = byf.get(fp, 0) + s
    print("   ", {k: round(100 * x / tot, 1) for k, x in byf.items()})
    for s, fp, ln, src in sorted(v, reverse=True)[:top]:
        print("   %5.1f%% %s:%d %s" % (100 * s / tot, fp, ln, src.strip()))
