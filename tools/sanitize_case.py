"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck) on the
GPU box: the C1 manifold (tiers 0-3, reduced / full / two-sided), a 64-env C4
slice (the TMA-staged face kernel: small chunks stage), a 256-env C5 slice,
sdf_eval with every output and the shape-parameter VJP."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_17538_b200 import binding, synth


def run_manifold(sc, tiers=(2,), modes=(0,)):
    S = binding.Scene(sc.shapes, sc.smooth)
    pairs = torch.from_numpy(sc.pairs).cuda()
    poses = torch.from_numpy(sc.poses).cuda()
    for mode in modes:
        offs = S.manifold_offsets(pairs, mode)
        C = S.manifold_size(sc.pairs, mode)
        for t in tiers:
            S.contact_manifold(pairs, offs, C, poses, t, mode=mode)
    torch.cuda.synchronize()
    return S


run_manifold(synth.c1_scene(), tiers=(0, 1, 2, 3), modes=(0, binding.FULL_MODE, binding.TWO_SIDED))
run_manifold(synth.c4_scene(64))
S = run_manifold(synth.c5_scene(256))
sc = synth.sdf_scene(64, 64)
S2 = binding.Scene(sc.shapes, sc.smooth)
ids = torch.from_numpy(sc.point_shapes).cuda()
po = torch.from_numpy(sc.point_poses).cuda()
pt = torch.from_numpy(sc.points).cuda()
S2.sdf_eval(ids, po, pt, sc.P, 31)
w = torch.ones(len(sc.points), device="cuda")
S2.sdf_param_grad(ids, po, pt, sc.P, w=w)
torch.cuda.synchronize()
print("sanitize case done")
