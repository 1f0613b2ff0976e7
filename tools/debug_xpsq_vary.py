"""Debug: GPU Hessian vs FD of the GPU gradient at the failing xpsq_vary points."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from oracle import oracle as O
from helpers import scene_of, pose8, unpack_sym3
from paper_2604_17538_b200 import synth, binding
import parity as PT
import test_gpu_parity as T
name, root = T._sdf_shapes()[8]
sc = scene_of([synth.make_shape(name, root)], ell=1.0)
osc = O.OracleScene(sc)
S = binding.Scene(sc.shapes, sc.smooth)
rng = np.random.default_rng(108)
B, P = 7, 333
poses = np.stack([pose8(rng.uniform(-0.1, 0.1, 3), synth.random_quats(rng, 1)[0]) for _ in range(B)]).astype(np.float32)
loc = rng.uniform(-0.45, 0.45, (B, P, 3))
pts = np.concatenate([loc[b] @ synth.quat_to_mat(poses[b, 3:7]).T + poses[b, :3] for b in range(B)]).astype(np.float32)
for n in [542, 596, 910]:
    b = n // P
    x = pts[n]
    h = 1e-3
    X = np.stack([x] + [x + s * h * np.eye(3)[i] for i in range(3) for s in (1, -1)]).astype(np.float32)
    ids = np.zeros(len(X), np.int32)
    po = np.repeat(poses[b:b + 1], len(X), 0)
    g = PT.gpu_sdf(S, ids, po, X, 1, 7)
    H = unpack_sym3(g["hess"][:, 0])
    Hf = np.stack([(g["grad"][:, 1 + 2 * i] - g["grad"][:, 2 + 2 * i]) / (2 * h) for i in range(3)], 1)
    o = osc.sdf_eval(np.array([0]), poses[b:b + 1], x[None].astype(np.float64), 1)
    Ho = unpack_sym3(o["hess"][0])
    print(n, "gpuH-oracle", np.abs(H - Ho).max(), "fdgpu-oracle", np.abs(Hf - Ho).max(), "gpuH-fdgpu", np.abs(H - Hf).max())
    print("  H", H[0], "\n  Ho", Ho[0], "\n  Hf", Hf[0])
