"""Parity helpers: run the CUDA path (through the C ABI binding) and the FP64
oracle on the same seeded inputs and compare them element by element with the
tolerances of BASELINE.json's north star:

  distances, depths, points          |err| <= 1e-5 max(|ref|, ell)
  q = W pbar (compact J)              the W tolerance x |pbar| + 1e-5 max(|ref|, ell)
  gradients, normals, W, d/dq, d/dpose |err| <= 1e-4 max(|ref|_inf, 1)
  Hessians, dn/dq, pose Hessians       |err| <= 1e-3 max(|ref|_inf, 1/ell)
  dom_idx                              identical unless the best two candidate
                                       depths are within 1e-4 ell (near tie)

Condition-aware exclusion: an element whose FP64 oracle value
moves by more than tol/10 when the FP32 inputs are perturbed by a relative
2^-24 is excluded and counted (the FP32 path cannot resolve it); the excluded
fraction is returned and must stay below 1%.
"""
from __future__ import annotations

import numpy as np

REL_EPS = 2.0 ** -24


def perturb_inputs(rng, poses, points=None):
    p = poses.astype(np.float64) * (1.0 + REL_EPS * rng.choice([-1.0, 1.0], poses.shape))
    if points is None:
        return p
    x = points.astype(np.float64) * (1.0 + REL_EPS * rng.choice([-1.0, 1.0], points.shape))
    return p, x


def tol_value(ref, ell):
    return 1e-5 * np.maximum(np.abs(ref), ell)


def tol_vec(ref, axis):
    return 1e-4 * np.maximum(np.abs(ref).max(axis=axis, keepdims=True), 1.0)


def tol_hess(ref, axis, ell):
    return 1e-3 * np.maximum(np.abs(ref).max(axis=axis, keepdims=True), 1.0 / ell)


def compare(name, got, ref, ref_pert, tol, report):
    """got/ref/ref_pert same shape; tol broadcastable.  Returns #failures."""
    got = np.asarray(got, dtype=np.float64)
    sens = np.abs(ref - ref_pert)
    excl = sens > tol / 10.0
    # non-finite values on either side are failures, never exclusions
    bad = ((np.abs(got - ref) > tol) & ~excl) | ~np.isfinite(got) | ~np.isfinite(ref)
    nb = int(bad.sum())
    report.append(dict(field=name, n=int(ref.size), excluded=int(excl.sum()), failures=nb,
                       max_err_over_tol=float(np.nanmax(np.where(excl, 0, np.abs(got - ref) / tol)))
                       if ref.size else 0.0))
    if nb:
        idx = np.argwhere(bad)[:5]
        report[-1]["examples"] = [(tuple(int(v) for v in i), float(got[tuple(i)]), float(ref[tuple(i)]))
                                  for i in idx]
    return nb


def gpu_manifold(scene, tier=2, pairs=None, poses=None, S=None, mode=0):
    import torch
    from paper_2604_17538_b200 import binding
    S = S or binding.Scene(scene.shapes, scene.smooth)
    pairs_np = scene.pairs if pairs is None else pairs
    poses_np = scene.poses if poses is None else poses
    pairs_t = torch.from_numpy(np.ascontiguousarray(pairs_np, dtype=np.int32)).cuda()
    poses_t = torch.from_numpy(np.ascontiguousarray(poses_np, dtype=np.float32)).cuda()
    offs = S.manifold_offsets(pairs_t, mode)
    C = S.manifold_size(pairs_np, mode)
    out = S.contact_manifold(pairs_t, offs, C, poses_t, tier, mode=mode)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["offsets"] = offs.cpu().numpy()
    res["C"] = C
    return res, S


def manifold_parity(scene, osc, gpu, tier, pair_idx, rng, ell, mode=0):
    """Compares the GPU manifold rows of pairs `pair_idx` (GPU ran the whole
    scene.pairs) with the oracle on those pairs.  Returns (failures, report)."""
    pairs = scene.pairs[pair_idx]
    ref = osc.contact_manifold(pairs=pairs, poses=scene.poses, mode=mode)
    refp = osc.contact_manifold(pairs=pairs, poses=perturb_inputs(rng, scene.poses), mode=mode)
    rows = np.concatenate([np.arange(gpu["offsets"][i], gpu["offsets"][i] + (ref["offsets"][k + 1] - ref["offsets"][k]))
                           for k, i in enumerate(pair_idx)]).astype(np.int64)
    rep = []
    nf = 0
    g = lambda k: gpu[k][..., rows]
    nf += compare("depth", g("depth"), ref["depth"], refp["depth"], tol_value(ref["depth"], ell), rep)
    nf += compare("point", g("point").T, ref["point"], refp["point"], tol_value(ref["point"], ell), rep)
    nf += compare("normal", g("normal").T, ref["normal"], refp["normal"], tol_vec(ref["normal"], 1), rep)
    if tier >= 1:
        nf += compare("W", g("W"), ref["W"], refp["W"], 1e-4 * np.maximum(np.abs(ref["W"]), 1.0), rep)
        # q = W pbar (pbar = q / W the gated contact point): its tolerance is
        # the W tolerance carried through |pbar| plus the point tolerance
        # (near a gate centre W moves by up to 1e-4 while q's own value
        # tolerance 1e-5 ell would not admit the same relative change)
        tW = 1e-4 * np.maximum(np.abs(ref["W"]), 1.0)
        pbar = np.abs(ref["q"]) / np.maximum(np.abs(ref["W"]), 1e-30)[:, None]
        tq = tol_value(ref["q"], ell) + tW[:, None] * np.minimum(pbar, 1e3 * ell)
        nf += compare("q", g("q").T, ref["q"], refp["q"], tq, rep)
    if tier >= 2:
        nf += compare("ddepth", g("ddepth").T, ref["ddepth"], refp["ddepth"], tol_vec(ref["ddepth"], 1), rep)
        dn = g("dnormal").reshape(3, 12, -1).transpose(2, 0, 1)
        nf += compare("dnormal", dn, ref["dnormal"], refp["dnormal"], tol_hess(ref["dnormal"], (1, 2), ell), rep)
    if tier >= 3:
        # second derivatives (f3): Hessian tolerance against the oracle's
        # second-order q-jets, condition-aware like every other field
        r2 = osc.manifold_d2depth(pairs=pairs, poses=scene.poses, mode=mode)
        r2p = osc.manifold_d2depth(pairs=pairs, poses=perturb_inputs(rng, scene.poses), mode=mode)
        nf += compare("d2depth", g("d2depth").T, r2, r2p, tol_hess(r2, 1, ell), rep)
    # dominant candidate, outside near ties of the two deepest candidates
    # (full mode: the candidate kind, compared exactly)
    ds = np.sort(ref["dcand"], axis=1)
    clear = (ds[:, 1] - ds[:, 0]) > 1e-4 * ell if not (mode & 4) else np.ones(len(ds), bool)
    dom_bad = int(((g("dom").astype(np.int64) != ref["dom"]) & clear).sum())
    rep.append(dict(field="dom", n=int(len(clear)), excluded=int((~clear).sum()), failures=dom_bad))
    nf += dom_bad
    return nf, rep


def gpu_sdf(S, shape_ids, poses, points, P, flags):
    import torch
    ids = torch.from_numpy(np.ascontiguousarray(shape_ids, dtype=np.int32)).cuda()
    po = torch.from_numpy(np.ascontiguousarray(poses, dtype=np.float32)).cuda()
    pt = torch.from_numpy(np.ascontiguousarray(points, dtype=np.float32)).cuda()
    out = S.sdf_eval(ids, po, pt, P, flags)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def sdf_parity(osc, gpu, shape_ids, poses, points, P, rng, ell):
    ref = osc.sdf_eval(shape_ids, poses, points, P, want_pose=True)
    pp, xp = perturb_inputs(rng, poses, points)
    refp = osc.sdf_eval(shape_ids, pp, xp, P, want_pose=True)
    rep = []
    nf = 0
    nf += compare("d", gpu["d"], ref["d"], refp["d"], tol_value(ref["d"], ell), rep)
    if "grad" in gpu:
        nf += compare("grad", gpu["grad"].T, ref["grad"], refp["grad"], tol_vec(ref["grad"], 1), rep)
    if "hess" in gpu:
        nf += compare("hess", gpu["hess"].T, ref["hess"], refp["hess"], tol_hess(ref["hess"], 1, ell), rep)
    if "dpose" in gpu:
        nf += compare("dpose", gpu["dpose"].T, ref["dpose"], refp["dpose"], tol_vec(ref["dpose"], 1), rep)
    if "d2pose" in gpu:
        nf += compare("d2pose", gpu["d2pose"].T, ref["d2pose"], refp["d2pose"], tol_hess(ref["d2pose"], 1, ell), rep)
        nf += compare("dxdpose", gpu["dxdpose"].T, ref["dxdpose"], refp["dxdpose"],
                      tol_hess(ref["dxdpose"], 1, ell), rep)
    return nf, rep


def excluded_fraction(rep):
    n = sum(r["n"] for r in rep)
    e = sum(r["excluded"] for r in rep)
    return e / max(n, 1)


def gpu_manifold_sampled(scene, pair_idx, tier=2):
    """Runs the whole scene on the GPU (bench launch configuration) and
    returns only the rows of pairs `pair_idx`, gathered on the device, in the
    layout of gpu_manifold (offsets re-based to the gathered rows)."""
    import torch
    from paper_2604_17538_b200 import binding
    S = binding.Scene(scene.shapes, scene.smooth)
    pairs_t = torch.from_numpy(np.ascontiguousarray(scene.pairs, dtype=np.int32)).cuda()
    poses_t = torch.from_numpy(np.ascontiguousarray(scene.poses, dtype=np.float32)).cuda()
    offs = S.manifold_offsets(pairs_t)
    C = S.manifold_size(scene.pairs)
    out = S.contact_manifold(pairs_t, offs, C, poses_t, tier)
    torch.cuda.synchronize()
    offs_h = offs.cpu().numpy()
    F = np.array([S.counts(int(a))[2] for a in scene.pairs[pair_idx, 3]])
    rows = np.concatenate([np.arange(offs_h[i], offs_h[i] + f) for i, f in zip(pair_idx, F)])
    rows_t = torch.from_numpy(rows).cuda()
    res = {k: v.index_select(v.dim() - 1, rows_t).cpu().numpy() for k, v in out.items()}
    del out
    torch.cuda.empty_cache()
    # re-based offsets: gathered pair k occupies [new_off[k], new_off[k] + F_k)
    full_offs = np.zeros(len(scene.pairs), np.int64)
    full_offs[pair_idx] = np.concatenate([[0], np.cumsum(F)[:-1]])
    res["offsets"] = full_offs
    res["C"] = int(len(rows))
    return res
