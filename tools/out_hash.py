"""Per-field SHA-1 of the manifold outputs of a workload set (GPU box), for
bitwise A/B checks between library builds (XPSQCM_LIB selects the build):

  XPSQCM_LIB=exp/lib_x.so python tools/out_hash.py > a.json
"""
import hashlib
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_17538_b200 import binding, synth  # noqa: E402

CASES = [("C1", lambda: synth.c1_scene()), ("C5s", lambda: synth.c5_scene(48)), ("C4s", lambda: synth.c4_scene(2)),
         ("C5", lambda: synth.c5_scene(1 << 16)), ("C4", lambda: synth.c4_scene(256)),
         ("C2", lambda: synth.c2_scene()), ("C3", lambda: synth.c3_scene(512))]
rep = {}
for name, mk in CASES:
    sc = mk()
    S = binding.Scene(sc.shapes, sc.smooth)
    pairs = torch.from_numpy(sc.pairs).cuda()
    poses = torch.from_numpy(sc.poses).cuda()
    offs = S.manifold_offsets(pairs)
    C = S.manifold_size(sc.pairs)
    for tier in (0, 1, 2):
        for mode in (0, binding.FULL_MODE, binding.TWO_SIDED):
            try:
                C2 = S.manifold_size(sc.pairs, mode) if mode else C
            except binding.CMError:
                continue   # e.g. two-sided with a half-space (no sampled surface)
            o2 = S.manifold_offsets(pairs, mode) if mode else offs
            out = S.contact_manifold(pairs, o2, C2, poses, tier, mode=mode)
            torch.cuda.synchronize()
            for k, v in out.items():
                rep["%s/t%d/m%d/%s" % (name, tier, mode, k)] = hashlib.sha1(v.cpu().numpy().tobytes()).hexdigest()
print(json.dumps(rep, indent=0, sort_keys=True))
