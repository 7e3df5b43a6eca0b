"""fp64 oracle of the neural-Gaussian decode.

TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py): only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this; it
shares no code with the CUDA path.

What it computes (§III-A "Scene Reconstruction": the final 2DGS
attributes {mu, R, S, rho, r, alpha} of each neural Gaussian are inferred by
passing the anchor features through the corresponding MLP; Scaffold-GS-style
anchors).  The paper fixes no sizes; the readings N1-N8 of
DESIGN.md §12 (from SPEC.md's design decisions) are:

  N1  anchor a: position x (fp32 [3]), feature f (F = 32, stored fp16),
      base scale l (fp32 [3], > 0); k = 5 neural Gaussians per anchor.
  N2  one MLP per head, two hidden layers of width 32 with ReLU:
          MLP(x) = W3 relu(W2 relu(W1 x + b1) + b2) + b3,
      weights stored fp16, biases fp32.  Geometry heads (offset, scale,
      rotation) read f; appearance heads (opacity, colour / intensity,
      ray-drop) read [f, d] with d = normalize(x - o), o = the sensor origin.
  N3  mu_j = x + O_j * l (elementwise);  s_j = (l_0 exp(S_j0), l_1 exp(S_j1)).
  N4  rotation: 6D (a1, a2) -> t_u = a1/|a1|, t_v = normalize(a2 - (t_u.a2) t_u),
      n = t_u x t_v (Gram-Schmidt).
  N5  opacity = sigmoid(.); camera colour c = sigmoid(.) (written to the
      surfel set as the degree-0 SH coefficient (c - 1/2)/C0, C0 = 1/(2 sqrt(pi)),
      which gs_project evaluates back to c); LiDAR intensity = sigmoid(.),
      ray-drop logit = the raw output.
  N6  surfel 5a + j comes from anchor a, output slot j.

Precision (the GPU's, not the oracle's): fp16 features and weights are exact
inputs here (promoted to fp64); the GPU rounds the view direction and every
hidden activation to fp16 (unit roundoff u = 2^-11) and accumulates in fp32.
`decode` returns, next to each fp64 value, a first-order bound of the error
those roundings can cause (propagated layer by layer with |W|), which the
parity test uses as its tolerance.
"""
from __future__ import annotations

import math

import numpy as np

K = 5
F = 32
HIDDEN = 32
U16 = 2.0 ** -11     # fp16 unit roundoff
U32 = 2.0 ** -24     # fp32 unit roundoff
C0 = 1.0 / (2.0 * math.sqrt(math.pi))

CAMERA_HEADS = ("offset", "scale", "rotation", "opacity", "color")
LIDAR_HEADS = ("offset", "scale", "rotation", "opacity", "intensity", "raydrop")
GEOMETRY = ("offset", "scale", "rotation")
OUT_DIM = {"offset": 3 * K, "scale": 2 * K, "rotation": 6 * K, "opacity": K, "color": 3 * K,
           "intensity": K, "raydrop": K}


def heads_of(modality: str):
    return CAMERA_HEADS if modality == "camera" else LIDAR_HEADS


def in_dim(head: str) -> int:
    return F if head in GEOMETRY else F + 3


def _mlp(x, ex, p):
    """One head on inputs x [n, in] (fp64) with per-element input error
    bounds ex [n, in].  Returns (z3 [n, out], bound [n, out])."""
    W1, b1, W2, b2, W3, b3 = (np.asarray(p[k], np.float64) for k in ("W1", "b1", "W2", "b2", "W3", "b3"))
    z1 = x @ W1.T + b1
    h1 = np.maximum(z1, 0.0)
    e1 = np.abs(ex) @ np.abs(W1).T + x.shape[1] * U32 * (np.abs(x) @ np.abs(W1).T + np.abs(b1))
    e1 = e1 + U16 * (h1 + e1)                       # relu is 1-Lipschitz; h1 rounded to fp16
    z2 = h1 @ W2.T + b2
    h2 = np.maximum(z2, 0.0)
    e2 = e1 @ np.abs(W2).T + HIDDEN * U32 * (h1 @ np.abs(W2).T + np.abs(b2))
    e2 = e2 + U16 * (h2 + e2)
    z3 = h2 @ W3.T + b3
    e3 = e2 @ np.abs(W3).T + HIDDEN * U32 * (h2 @ np.abs(W3).T + np.abs(b3))
    return z3, e3


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def decode(position, feature, base_scale, decoder: dict, view_origin, modality: str = "camera"):
    """position [n,3] f32, feature [n,32] f16, base_scale [n,3] f32, decoder
    {head: {W1, b1, W2, b2, W3, b3}} (fp16 weights, fp32 biases), view_origin
    [3] -> dict of fp64 surfel attributes for the n*K surfels (surfel 5a+j)
    and their error bounds ("<name>_tol")."""
    x = np.asarray(position, np.float64)
    f = np.asarray(feature, np.float16).astype(np.float64)
    l = np.asarray(base_scale, np.float64)
    o = np.asarray(view_origin, np.float64)
    n = x.shape[0]
    v = x - o
    d = v / np.linalg.norm(v, axis=1, keepdims=True)
    xin_g, ein_g = f, np.zeros_like(f)
    xin_a = np.concatenate([f, d], axis=1)
    ein_a = np.concatenate([np.zeros_like(f), (U16 + 8 * U32) * np.abs(d) + 4 * U32], axis=1)
    z, e = {}, {}
    for h in heads_of(modality):
        xi, ei = (xin_g, ein_g) if h in GEOMETRY else (xin_a, ein_a)
        z[h], e[h] = _mlp(xi, ei, decoder[h])
    out = {}
    # N3: centres and scales
    O = z["offset"].reshape(n, K, 3)
    eO = e["offset"].reshape(n, K, 3)
    mu = x[:, None, :] + O * l[:, None, :]
    out["means"] = mu.reshape(n * K, 3)
    out["means_tol"] = (eO * l[:, None, :] + 4 * U32 * (np.abs(x)[:, None, :] + np.abs(O * l[:, None, :]))
                        ).reshape(n * K, 3)
    S = z["scale"].reshape(n, K, 2)
    eS = e["scale"].reshape(n, K, 2)
    s = l[:, None, :2] * np.exp(S)
    out["scales"] = s.reshape(n * K, 2)
    out["scales_tol"] = (s * (np.expm1(eS) + 8 * U32)).reshape(n * K, 2)
    # N4: rotation frame
    R6 = z["rotation"].reshape(n, K, 6)
    eR = e["rotation"].reshape(n, K, 6)
    a1, a2 = R6[..., :3], R6[..., 3:]
    da1, da2 = np.linalg.norm(eR[..., :3], axis=-1), np.linalg.norm(eR[..., 3:], axis=-1)
    n1 = np.linalg.norm(a1, axis=-1)
    tu = a1 / n1[..., None]
    b = a2 - np.sum(tu * a2, axis=-1, keepdims=True) * tu
    nb = np.linalg.norm(b, axis=-1)
    tv = b / nb[..., None]
    nn = np.cross(tu, tv)
    etu = 2.0 * da1 / n1
    eb = 2.0 * da2 + 2.0 * np.linalg.norm(a2, axis=-1) * etu
    etv = 2.0 * eb / nb
    out["frame"] = np.stack([tu, tv, nn], axis=-1).reshape(n * K, 3, 3)   # columns t_u, t_v, n
    out["frame_tol"] = (np.stack([etu, etv, etu + etv], axis=-1) + 1e-6).reshape(n * K, 3)
    # N5: opacity and radiometry
    out["opacities"] = _sigmoid(z["opacity"]).reshape(n * K)
    out["opacities_tol"] = (0.25 * e["opacity"] + 4 * U32).reshape(n * K)
    if modality == "camera":
        c = _sigmoid(z["color"]).reshape(n * K, 3)
        out["sh_dc"] = (c - 0.5) / C0
        out["sh_dc_tol"] = ((0.25 * e["color"] + 4 * U32).reshape(n * K, 3) / C0 + 8 * U32 * np.abs(out["sh_dc"]))
    else:
        out["intensity"] = _sigmoid(z["intensity"]).reshape(n * K)
        out["intensity_tol"] = (0.25 * e["intensity"] + 4 * U32).reshape(n * K)
        out["raydrop_logit"] = z["raydrop"].reshape(n * K)
        out["raydrop_logit_tol"] = (e["raydrop"] + 4 * U32 * np.abs(z["raydrop"])).reshape(n * K)
    return out


def dense_loop(x, W, b):
    """y_i = b_i + sum_j W_ij x_j with explicit Python loops (the independent
    brute-force formulation the numpy layers are pinned against)."""
    out = []
    for row in range(len(W)):
        acc = float(b[row])
        for j in range(len(x)):
            acc += float(W[row][j]) * float(x[j])
        out.append(acc)
    return out
