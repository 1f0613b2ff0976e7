"""Test helpers: building small scenes from shape descriptions, pose
perturbations for finite differences.  No arithmetic of the method."""
import math

import numpy as np

from paper_2604_17538_b200 import synth


def scene_of(shapes, ell=1.0, pairs=None, poses=None, **smooth_over):
    sp = synth.smooth_params(ell)
    sp.update(smooth_over)
    if pairs is None:
        pairs = np.zeros((0, 5), np.int32)
    if poses is None:
        poses = np.zeros((1, 1, 8), np.float32)
        poses[0, 0, 3] = 1.0
    return synth.Scene("test", shapes, sp, np.asarray(pairs, np.int32), np.asarray(poses, np.float32), ell)


def pose8(t=(0, 0, 0), q=(1, 0, 0, 0)):
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q)
    return np.array([t[0], t[1], t[2], q[0], q[1], q[2], q[3], 0.0])


def rot_exp_quat(w):
    w = np.asarray(w, dtype=np.float64)
    th = np.linalg.norm(w)
    if th == 0.0:
        return np.array([1.0, 0, 0, 0])
    return synth.quat_from_axis_angle(w / th, th)


def perturb(p8, dq):
    """World-frame left perturbation: t <- t + dt, R <- exp([w]x) R."""
    p = np.array(p8, dtype=np.float64)
    p[:3] += dq[:3]
    p[3:7] = synth.quat_mul(rot_exp_quat(dq[3:6]), p[3:7])
    return p


def rand_pose(rng, scale=0.3):
    return pose8(rng.uniform(-scale, scale, 3), synth.random_quats(rng, 1)[0])


def skew(v):
    return np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])


HIDX = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def unpack_sym3(h6):
    H = np.zeros((3, 3))
    for k, (i, j) in enumerate(HIDX):
        H[i, j] = H[j, i] = h6[k]
    return H


def unpack_sym6(h21):
    H = np.zeros((6, 6))
    k = 0
    for i in range(6):
        for j in range(i, 6):
            H[i, j] = H[j, i] = h21[k]
            k += 1
    return H
