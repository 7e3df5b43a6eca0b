"""NumPy naive renderer with a DIFFERENT intersection formulation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Used to cross-check the
C oracle on small scenes.  Where oracle.c intersects the ray's plane pair
(Eq. 2), this file intersects the ray with the surfel's own plane:

    t = (n . mu_s) / (n . d),   P = t d,   u = t_u.(P - mu_s) / s_u,
                                          v = t_v.(P - mu_s) / s_v,

and takes the SH basis from scipy's complex spherical harmonics
(scipy.special.sph_harm_y, Condon-Shortley phase) instead of hand-written
constants.  Fisheye rays are inverted by Newton's method instead of bisection.
Everything else follows DESIGN.md §2 literally; fp64 throughout.  Vectorised
over surfels, one ray at a time: only for small inputs.
"""
from __future__ import annotations

import numpy as np
import scipy.special as sps

DEFAULTS = dict(near=0.2, alpha_max=0.99, alpha_min=1.0 / 255.0, t_min=1e-4, support_rho=9.0,
                lowpass_sigma=1.0 / np.sqrt(2.0), bg_rgb=(0.0, 0.0, 0.0), bg_range=0.0,
                bg_raydrop=1.0)


def _rot(q):
    q = q.astype(np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z); R[:, 0, 1] = 2 * (x * y - w * z); R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z); R[:, 1, 1] = 1 - 2 * (x * x + z * z); R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y); R[:, 2, 1] = 2 * (y * z + w * x); R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def sh_basis_scipy(dirs, degree):
    """3DGS real SH basis: sqrt2*Im(Y_l^|m|) (m<0), Y_l^0, sqrt2*Re(Y_l^m) (m>0)
    with scipy's complex Y_l^m (Condon-Shortley phase included)."""
    th = np.arccos(np.clip(dirs[:, 2], -1, 1))
    ph = np.arctan2(dirs[:, 1], dirs[:, 0])
    cols = []
    for l in range(degree + 1):
        for m in range(-l, l + 1):
            c = sps.sph_harm_y(l, abs(m), th, ph)
            cols.append(np.sqrt(2) * c.imag if m < 0 else (c.real if m == 0 else np.sqrt(2) * c.real))
    return np.stack(cols, axis=1)


def _kb(k, th):
    t2 = th * th
    return th * (1 + k[0] * t2 + k[1] * t2 ** 2 + k[2] * t2 ** 3 + k[3] * t2 ** 4)


def _kb_inv_newton(k, td, theta_max):
    th = min(td, theta_max)
    for _ in range(100):
        t2 = th * th
        f = _kb(k, th) - td
        df = 1 + 3 * k[0] * t2 + 5 * k[1] * t2 ** 2 + 7 * k[2] * t2 ** 3 + 9 * k[3] * t2 ** 4
        nxt = min(max(th - f / df, 0.0), theta_max)
        if abs(nxt - th) < 1e-16:
            break
        th = nxt
    return th


def _ray(se, col, row):
    """direction d (pinhole: z=1; else unit), pixel p, validity"""
    p = np.array([col + 0.5, row + 0.5])
    if se.kind == 0:
        return np.array([(p[0] - se.cx) / se.fx, (p[1] - se.cy) / se.fy, 1.0]), p, True
    if se.kind == 1:
        k = np.asarray(se.k, np.float64)
        m = np.array([(p[0] - se.cx) / se.fx, (p[1] - se.cy) / se.fy])
        td = np.hypot(m[0], m[1])
        tdmax = _kb(k, float(se.theta_max))
        th = _kb_inv_newton(k, min(td, tdmax), float(se.theta_max))
        psi = np.arctan2(m[1], m[0]) if td > 0 else 0.0
        d = np.array([np.sin(th) * np.cos(psi), np.sin(th) * np.sin(psi), np.cos(th)])
        return d, p, td <= tdmax
    if se.kind == 3:   # cylindrical (Eq. 4): azimuth about y, height over the y-axis distance
        phi = (p[0] - se.cx) / se.fx
        return np.array([np.sin(phi), (p[1] - se.cy) / se.fy, np.cos(phi)]), p, True
    th = float(se.beam_elevation[row])
    ph = float(se.azimuth0) + col * float(se.azimuth_step)
    return np.array([np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), np.sin(th)]), p, True


def _prep(s, se, o):
    W = np.asarray(se.world_to_sensor, np.float64)
    Rs, ts = W[:, :3], W[:, 3]
    mu = s.means.astype(np.float64)
    # pinned-order sensor-frame centre (reading R9): ((a+b)+c)+t, no FMA in numpy
    mus = np.stack([((Rs[k, 0] * mu[:, 0] + Rs[k, 1] * mu[:, 1]) + Rs[k, 2] * mu[:, 2]) + ts[k]
                    for k in range(3)], axis=1)
    if se.kind == 0:
        key = mus[:, 2].astype(np.float32)
    else:
        key = np.sqrt((mus[:, 0] * mus[:, 0] + mus[:, 1] * mus[:, 1]) + mus[:, 2] * mus[:, 2]).astype(np.float32)
    culled = ~(key >= np.float32(o["near"])) | ~np.isfinite(key)
    R = _rot(s.quats)
    tu = np.einsum("ij,nj->ni", Rs, R[:, :, 0])
    tv = np.einsum("ij,nj->ni", Rs, R[:, :, 1])
    nn = np.einsum("ij,nj->ni", Rs, R[:, :, 2])
    side = np.sum(nn * mus, axis=1)
    ns = np.where(side[:, None] > 0, -nn, nn)
    su, sv = s.scales[:, 0].astype(np.float64), s.scales[:, 1].astype(np.float64)
    if se.kind == 0:
        c = np.stack([se.fx * mus[:, 0] / mus[:, 2] + se.cx, se.fy * mus[:, 1] / mus[:, 2] + se.cy], 1)
        cdepth = mus[:, 2]
    elif se.kind == 1:
        k = np.asarray(se.k, np.float64)
        rxy = np.hypot(mus[:, 0], mus[:, 1])
        th = np.arctan2(rxy, mus[:, 2])
        td = _kb(k, th)
        safe = np.where(rxy > 0, rxy, 1.0)
        c = np.stack([np.where(rxy > 0, se.cx + se.fx * td * mus[:, 0] / safe, se.cx),
                      np.where(rxy > 0, se.cy + se.fy * td * mus[:, 1] / safe, se.cy)], 1)
        cdepth = np.linalg.norm(mus, axis=1)
    elif se.kind == 3:
        c = np.stack([se.cx + se.fx * np.arctan2(mus[:, 0], mus[:, 2]),
                      se.cy + se.fy * mus[:, 1] / np.hypot(mus[:, 0], mus[:, 2])], 1)
        cdepth = np.linalg.norm(mus, axis=1)
    else:
        c = np.zeros((s.n, 2))
        cdepth = np.linalg.norm(mus, axis=1)
    if se.kind == 2:
        val = np.stack([s.intensity.astype(np.float64),
                        1.0 / (1.0 + np.exp(-s.raydrop_logit.astype(np.float64))),
                        np.zeros(s.n)], 1)
    else:
        o_w = -Rs.T @ ts
        v = mu - o_w
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        B = sh_basis_scipy(v, s.sh_degree)
        val = np.maximum(np.einsum("nj,njc->nc", B, s.sh.astype(np.float64)) + 0.5, 0.0)
    return dict(mus=mus, key=key, culled=culled, tu=tu, tv=tv, ns=ns, nn=nn, su=su, sv=sv, c=c,
                cdepth=cdepth, val=val, o=s.opacities.astype(np.float64))


def render(s, se, rays=None, **opts):
    """Returns out [n_rays, 8] in the same channel layout as oracle.render."""
    o = dict(DEFAULTS)
    o.update(opts)
    P = _prep(s, se, o)
    if rays is None:
        rays = np.arange(se.width * se.height)
    out = np.zeros((len(rays), 8))
    cam = se.kind != 2
    keybits = P["key"].view(np.uint32)
    for r, ray in enumerate(rays):
        col, row = int(ray % se.width), int(ray // se.width)
        d, p, valid = _ray(se, col, row)
        T, acc, D, Nr = 1.0, np.zeros(3), 0.0, np.zeros(3)
        if valid and s.n > 0:
            # ray / surfel-plane intersection
            nd = P["nn"] @ d
            with np.errstate(divide="ignore", invalid="ignore"):
                t = np.sum(P["nn"] * P["mus"], axis=1) / nd
                off = t[:, None] * d[None, :] - P["mus"]
                u = np.sum(P["tu"] * off, axis=1) / P["su"]
                v = np.sum(P["tv"] * off, axis=1) / P["sv"]
                rho3 = np.where(np.isfinite(u) & np.isfinite(v), u * u + v * v, np.inf)
            depth3 = t if se.kind == 0 else t * np.linalg.norm(d)
            if cam:
                rho2 = np.sum((p[None, :] - P["c"]) ** 2, axis=1) / o["lowpass_sigma"] ** 2
                use3 = rho3 <= rho2
                rho = np.where(use3, rho3, rho2)
                depth = np.where(use3, depth3, P["cdepth"])
            else:
                rho, depth = rho3, depth3
            with np.errstate(over="ignore", invalid="ignore"):
                alpha = np.minimum(o["alpha_max"], P["o"] * np.exp(-0.5 * rho))
                ok = (~P["culled"]) & (rho <= o["support_rho"]) & (depth >= o["near"]) & (alpha >= o["alpha_min"])
            idx = np.nonzero(ok)[0]
            order = idx[np.lexsort((idx, keybits[idx]))]
            for i in order:
                Tn = T * (1 - alpha[i])
                if Tn < o["t_min"]:
                    break
                w = alpha[i] * T
                acc += w * P["val"][i]
                Nr += w * P["ns"][i]
                D += w * depth[i]
                T = Tn
        A = 1.0 - T
        if cam:
            if not valid:
                out[r, :3] = o["bg_rgb"]
            else:
                out[r, :3] = acc + T * np.asarray(o["bg_rgb"])
                out[r, 3] = D / A if A > 0 else 0.0
                out[r, 4:7] = Nr
                out[r, 7] = A
        else:
            out[r, 0] = D / A if A > 0 else o["bg_range"]
            out[r, 1] = acc[0]
            out[r, 2] = acc[1] + T * o["bg_raydrop"]
            out[r, 3] = A
    return out
