"""Small shared helpers for tests: hand-built scenes and sensors (inputs only)."""
from __future__ import annotations

import json
import os

import numpy as np

import scenegen as sg

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def quat_from_R(R):
    """(w,x,y,z) of a rotation matrix whose columns are (t_u, t_v, n)."""
    return sg._quat_from_frame(R[None, :, 0], R[None, :, 1], R[None, :, 2])[0]


def scene(surfs, sh_degree=0):
    """surfs: list of dicts with mu, R (3x3, columns t_u,t_v,n) or quat, s (2), o,
    rgb (3) [, intensity, drop_logit]."""
    n = len(surfs)
    nc = (sh_degree + 1) ** 2
    means = np.zeros((n, 3)); quats = np.zeros((n, 4)); scales = np.zeros((n, 2))
    op = np.zeros(n); sh = np.zeros((n, nc, 3)); inten = np.zeros(n); drop = np.zeros(n)
    for i, s in enumerate(surfs):
        means[i] = s["mu"]
        quats[i] = s["quat"] if "quat" in s else quat_from_R(np.asarray(s.get("R", np.eye(3)), np.float64))
        scales[i] = s["s"]
        op[i] = s["o"]
        sh[i, 0] = (np.asarray(s.get("rgb", [0.5, 0.5, 0.5])) - 0.5) / sg.SH_C0
        inten[i] = s.get("intensity", 0.0)
        drop[i] = s.get("drop_logit", 0.0)
    f = lambda a: np.ascontiguousarray(a, np.float32)
    return sg.Surfels(f(means), f(quats), f(scales), f(op), f(sh), sh_degree, f(inten), f(drop))


def empty_scene(sh_degree=0):
    f = lambda *s: np.zeros(s, np.float32)
    return sg.Surfels(f(0, 3), f(0, 4), f(0, 2), f(0), f(0, (sh_degree + 1) ** 2, 3), sh_degree,
                      f(0), f(0))


def small_pinhole(w=32, h=24, f=20.0):
    return sg.pinhole(w, h, f, w / 2.0, h / 2.0, sg.identity_pose())


def small_lidar(h=8, w=64, top=10.0, bottom=-10.0):
    return sg.lidar64(sg.lidar_pose([0.0, 0.0, 0.0]), height=h, width=w, top_deg=top,
                      bottom_deg=bottom)


def random_small_scene(seed, n=24, lo=(-3, -3, 1), hi=(3, 3, 7), sh_degree=1):
    rng = np.random.default_rng(seed)
    return sg.random_surfels(rng, n, list(lo), list(hi), 0.05, 0.8, sh_degree=sh_degree,
                             lidar_attrs=True)
