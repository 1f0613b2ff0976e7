"""Determinism / non-finite diagnostic of the C5 manifold (GPU box)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_17538_b200 import binding, synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
wl = sys.argv[2] if len(sys.argv) > 2 else "C5"
sc = {"C5": lambda: synth.c5_scene(n), "C4": lambda: synth.c4_scene(n), "C3": lambda: synth.c3_scene(n),
      "C6": lambda: synth.c6_scene(n)}[wl]()
S = binding.Scene(sc.shapes, sc.smooth)
pairs = torch.from_numpy(sc.pairs).cuda()
poses = torch.from_numpy(sc.poses).cuda()
offs = S.manifold_offsets(pairs)
C = S.manifold_size(sc.pairs)
a = S.contact_manifold(pairs, offs, C, poses, 2)
b = S.contact_manifold(pairs, offs, C, poses, 2)
torch.cuda.synchronize()
offs_h = offs.cpu().numpy()
rep = {}
for k in a:
    x, y = a[k], b[k]
    if x.dtype == torch.float32:
        nf = (~torch.isfinite(x)).reshape(-1, C).any(0)
        bad = (x != y) & ~(torch.isnan(x) & torch.isnan(y))
        badc = bad.reshape(-1, C).any(0)
    else:
        nf = torch.zeros(C, dtype=torch.bool, device=x.device)
        badc = (x != y)
    rows_nf = torch.nonzero(nf).flatten().cpu().numpy()
    rows_bad = torch.nonzero(badc).flatten().cpu().numpy()
    pr_nf = np.unique(np.searchsorted(offs_h, rows_nf, side="right") - 1)
    pr_bad = np.unique(np.searchsorted(offs_h, rows_bad, side="right") - 1)
    rep[k] = {"nonfinite_rows": int(len(rows_nf)), "nonfinite_pairs": pr_nf[:20].tolist(),
              "mismatch_rows": int(len(rows_bad)), "mismatch_pairs": pr_bad[:20].tolist(),
              "shapes_nf": [(int(sc.pairs[p, 3]), int(sc.pairs[p, 4])) for p in pr_nf[:10]],
              "shapes_bad": [(int(sc.pairs[p, 3]), int(sc.pairs[p, 4])) for p in pr_bad[:10]]}
print(json.dumps(rep, indent=1))
