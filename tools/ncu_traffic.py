"""DRAM traffic and duration per manifold kernel of one chunk from an
`ncu --set full` capture (tools/profile_round.sh), and the per-pair DRAM
bytes of the whole chunk -> JSON (profiles/<round>_traffic_c5.json)."""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else "C5"
first_n = int(sys.argv[4]) if len(sys.argv) > 4 else 0   # only the first N kernels (one chunk)
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(txt))
h, units = rows[0], rows[1]
def col(r, k):
    v = r[h.index(k)].replace(",", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(units[h.index(k)], 1)
    return float(v) * scale
ks = []
grid = None
for r in (rows[2:2 + first_n] if first_n else rows[2:]):
    g = int(r[h.index("Grid Size")].strip("()").split(",")[0])
    grid = g if grid is None else max(grid, g)
    ks.append({"kernel": r[h.index("Kernel Name")].split("(")[0], "ns": col(r, "gpu__time_duration.sum"),
               "dram_read_bytes": col(r, "dram__bytes_read.sum"), "dram_write_bytes": col(r, "dram__bytes_write.sum")})
tot = sum(k["dram_read_bytes"] + k["dram_write_bytes"] for k in ks)
tns = sum(k["ns"] for k in ks)
for k in ks:
    k["share_of_chunk_time"] = k["ns"] / tns
res = {"workload": workload, "pairs": grid, "dram_read_bytes": sum(k["dram_read_bytes"] for k in ks),
       "dram_write_bytes": sum(k["dram_write_bytes"] for k in ks), "bytes_per_pair": tot / grid,
       "kernels": ks,
       "source": "%s (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum over the k_mf_* kernels of "
                 "the first %d-unit chunk of a %s shard; serialised, cold-cache replays)" % (rep, grid, workload)}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "kernels"}, indent=1))
for k in ks:
    print("%-32s %8.1f us  %5.1f%%  R %7.1f MB  W %7.1f MB" % (k["kernel"][-32:], k["ns"] / 1e3, 100 * k["share_of_chunk_time"],
                                                             k["dram_read_bytes"] / 1e6, k["dram_write_bytes"] / 1e6))
