"""Per-phase cycle split of k_contact_manifold (build with CM_PHASE_TIMING=1)."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("XPSQCM_LIB", os.path.join(ROOT, "exp/libxpsqcm_t.so"))
import torch
from paper_2604_17538_b200 import binding, synth
wl = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
sc = {"C5": lambda: synth.c5_scene(n), "C4": lambda: synth.c4_scene(n), "C3": lambda: synth.c3_scene(n),
      "C2": lambda: synth.c2_scene(n)}[wl]()
S = binding.Scene(sc.shapes, sc.smooth)
pairs = torch.from_numpy(sc.pairs).cuda(); poses = torch.from_numpy(sc.poses).cuda()
offs = S.manifold_offsets(pairs); Cn = S.manifold_size(sc.pairs)
out = S.alloc_manifold(Cn, 2, pairs.device)
L = binding.lib()
buf = (C.c_ulonglong * 20)()
L.cm_debug_phase_cycles(buf)
base = np.array(buf[:]).reshape(4, 5)
S.contact_manifold(pairs, offs, Cn, poses, 2, out); torch.cuda.synchronize()
L.cm_debug_phase_cycles(buf)
cyc = np.array(buf[:]).reshape(4, 5) - base
names = ["vertices", "traces", "midpoints", "faces", "prologue"]
for k, nm in enumerate(["SQ-flat", "XPSQ", "XPSQ-vary", "SQ-nested"]):
    t = cyc[k].sum()
    if t:
        print(wl, nm, " ".join("%s %.1f%%" % (names[i], 100 * cyc[k][i] / t) for i in range(5)), "total Gcyc %.2f" % (t / 1e9))
