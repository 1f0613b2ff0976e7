"""Locate non-finite manifold outputs of given C5 pairs (GPU box): full-mode
candidates, their points in the SDF body's frame, and sdf_eval there."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_17538_b200 import binding, synth

n = int(sys.argv[1])
pairs_idx = [int(x) for x in sys.argv[2].split(",")]
sc = synth.c5_scene(n)
S = binding.Scene(sc.shapes, sc.smooth)
out = {}
for pi in pairs_idx:
    pr = sc.pairs[pi:pi + 1].copy()
    pr[0, 0] = 0
    po = sc.poses[pi:pi + 1].copy()
    pt = torch.from_numpy(pr).cuda()
    pot = torch.from_numpy(po).cuda()
    res = {}
    for mode in (0, binding.FULL_MODE):
        offs = S.manifold_offsets(pt, mode)
        C = S.manifold_size(pr, mode)
        o = S.contact_manifold(pt, offs, C, pot, 2, mode=mode)
        torch.cuda.synchronize()
        o = {k: v.cpu().numpy() for k, v in o.items()}
        bad = set()
        for k, v in o.items():
            if v.dtype == np.float32:
                bad |= set(np.nonzero(~np.isfinite(v.reshape(-1, C)).any(0))[0].tolist())
        rows = sorted(bad)
        res["mode%d" % mode] = {"C": C, "bad_rows": rows[:20],
                                "bad": [{"row": r, "point": o["point"][:, r].tolist(), "depth": float(o["depth"][r]),
                                         "normal": o["normal"][:, r].tolist()} for r in rows[:6]]}
        if mode and rows:
            # SDF body pose (slot B = 1) and the candidate points in its frame
            pB = po[0, 1]
            R = synth.quat_to_mat(pB[3:7].astype(np.float64))
            pts = np.array([o["point"][:, r] for r in rows], np.float32)
            loc = (pts.astype(np.float64) - pB[:3]) @ R
            ids = torch.tensor([int(pr[0, 4])], dtype=torch.int32, device="cuda")
            g = S.sdf_eval(ids, torch.from_numpy(pB.reshape(1, 8)).cuda(), torch.from_numpy(pts).cuda(), len(pts),
                           binding.SDF_VALUE | binding.SDF_GRAD | binding.SDF_HESS)
            g = {k: v.cpu().numpy() for k, v in g.items()}
            res["sdf_eval_at_bad"] = {"local": loc.tolist(), "d": g["d"].tolist(), "grad": g["grad"].T.tolist(),
                                      "hess": g["hess"].T.tolist()}
    out[pi] = {"shapes": [int(pr[0, 3]), int(pr[0, 4])], **res}
print(json.dumps(out, indent=1))
