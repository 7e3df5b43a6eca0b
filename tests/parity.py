"""Tolerance protocol of DESIGN.md §5 (GPU vs oracle), shared by GPU tests,
smoke() and bench.py's parity spot check.

Every ray is held to the north_star tolerances (1e-4 absolute on colour,
alpha, normal, intensity, ray-drop; 1e-4 relative on depth and range):

  * a ray the oracle does not flag must match the oracle's composite;
  * a flagged ray (a near decision) must match one of the
    oracle's variants of that ray (oracle.variants: every composite the
    definition gives when each flagged pair takes each admissible state) on
    all channels at once; when one of its pairs is an ill-conditioned
    intersection (F_COND, alpha known only within an fp32 interval) it must
    lie, channel by channel, inside the envelope of the variants widened by
    the same tolerances.

A flagged ray is "ambiguous" when its admissible results differ from each
other by more than the tolerance (most flagged rays are not: e.g. a stop
decision at T ~ 1e-4 changes the result by less than T).  Ambiguous rays may
number at most MAX_AMBIGUOUS_FRAC of the rays (the pre-kernel flagged-ray
bound, 2e-3); unresolved rays (more variants than the oracle enumerates)
none.
"""
from __future__ import annotations

import numpy as np

import oracle

TOL_ABS = 1e-4        # colour, alpha, normal, intensity, raydrop (north_star)
TOL_REL = 1e-4        # depth, range (north_star)
MAX_AMBIGUOUS_FRAC = 2e-3
MAX_VARIANTS = 256


def sample_rays(sensor, n_random=4096, n_tiles=16, tile=16, seed=0):
    """All pixels of `n_tiles` random tiles plus `n_random` random pixels."""
    rng = np.random.default_rng(seed)
    W, H = sensor.width, sensor.height
    ntx, nty = (W + tile - 1) // tile, (H + tile - 1) // tile
    rays = []
    for t in rng.choice(ntx * nty, min(n_tiles, ntx * nty), replace=False):
        ty, tx = divmod(int(t), ntx)
        ys, xs = np.meshgrid(np.arange(ty * tile, min(H, ty * tile + tile)),
                             np.arange(tx * tile, min(W, tx * tile + tile)), indexing="ij")
        rays.append((ys * W + xs).ravel())
    rays.append(rng.choice(W * H, min(n_random, W * H), replace=False))
    return np.unique(np.concatenate(rays)).astype(np.int64)


def _channels(cam):
    # (absolute-tolerance channels, relative-tolerance channel, alpha channel)
    return ([0, 1, 2, 4, 5, 6, 7], 3, 7) if cam else ([1, 2, 3], 0, 3)


def _errors(g, r, cam):
    """Per-ray (max abs error over the absolute channels, relative error of
    depth/range, empty-rule violation) of g against r, both [..., C]."""
    abs_ch, rel_ch, a_ch = _channels(cam)
    err_abs = np.abs(g[..., abs_ch] - r[..., abs_ch]).max(axis=-1)
    has = r[..., a_ch] > 0
    rel = np.where(has, np.abs(g[..., rel_ch] - r[..., rel_ch]) / np.maximum(np.abs(r[..., rel_ch]), 1e-30), 0.0)
    empty_bad = (~has) & ((g[..., a_ch] != 0) | (g[..., rel_ch] != r[..., rel_ch]))
    return err_abs, rel, empty_bad


def _envelope_ok(g, var, cam):
    """g [C] inside the per-channel envelope of var [V, C] widened by the
    tolerances; a ray with alpha = 0 in every variant follows the empty rule."""
    abs_ch, rel_ch, a_ch = _channels(cam)
    lo, hi = var.min(axis=0), var.max(axis=0)
    if hi[a_ch] == 0:
        return bool(g[a_ch] == 0 and g[rel_ch] == var[0, rel_ch])
    ok = np.all((g[abs_ch] >= lo[abs_ch] - TOL_ABS) & (g[abs_ch] <= hi[abs_ch] + TOL_ABS))
    has = var[:, a_ch] > 0
    dl, dh = var[has, rel_ch].min(), var[has, rel_ch].max()
    return bool(ok and dl * (1 - TOL_REL) - 1e-30 <= g[rel_ch] <= dh * (1 + TOL_REL) + 1e-30)


def compare(gpu_chw: np.ndarray, ref: np.ndarray, flags: np.ndarray, rays: np.ndarray, sensor,
            surfels=None, opts=None):
    """gpu_chw: [C,H,W] GPU output; ref: [n,8] oracle output for `rays`;
    flags: the oracle's per-ray flags.  `surfels` (the scene) is needed to
    enumerate the variants of flagged rays; without it flagged rays fail.
    Returns a stats dict; stats['ok'] tells whether the gate passed."""
    W = sensor.width
    cam = sensor.kind != oracle.LIDAR
    C = 8 if cam else 4
    g = gpu_chw.reshape(C, -1)[:, rays].T.astype(np.float64)
    r = ref[:, :C]
    fl = flags != 0
    err_abs, rel, empty_bad = _errors(g, r, cam)
    bad = (~fl) & ((err_abs > TOL_ABS) | (rel > TOL_REL) | empty_bad)
    # flagged rays: two-sided, against the oracle's variants
    fidx = np.nonzero(fl)[0]
    bad_flagged = np.zeros(len(rays), bool)
    unresolved = 0
    ambiguous = 0
    n_cond = 0
    nominal_ok = 0
    if len(fidx):
        if surfels is None:
            bad_flagged[fidx] = True
        else:
            var, nvar, seen = oracle.variants(surfels, sensor, rays[fidx], MAX_VARIANTS, **(opts or {}))
            for k, i in enumerate(fidx):
                nv = int(nvar[k])
                if nv > MAX_VARIANTS:
                    unresolved += 1
                    bad_flagged[i] = True
                    continue
                v = var[k, :nv, :C]
                # ambiguous: the admissible results differ by more than the tolerance
                sa, sr, sb = _errors(v, v[:1].repeat(nv, 0), cam)
                ambiguous += bool(np.any((sa > TOL_ABS) | (sr > TOL_REL) | sb))
                ea, er, eb = _errors(g[i][None, :], v, cam)
                match = (ea <= TOL_ABS) & (er <= TOL_REL) & ~eb
                nominal_ok += bool(match[0])
                if seen[k] & oracle.F_COND:
                    n_cond += 1
                    bad_flagged[i] = not (match.any() or _envelope_ok(g[i], v, cam))
                else:
                    bad_flagged[i] = not match.any()
    uf = ~fl
    stats = dict(n=len(rays), flagged=int(fl.sum()), ambiguous=ambiguous, flagged_cond=n_cond,
                 unresolved=unresolved,
                 flagged_nominal_match=int(nominal_ok),
                 bad=int(bad.sum()), bad_flagged=int(bad_flagged.sum()),
                 max_abs_unflagged=float(err_abs[uf].max()) if uf.any() else 0.0,
                 p9999_abs=float(np.quantile(err_abs[uf], 0.9999)) if uf.any() else 0.0,
                 mean_abs=float(err_abs[uf].mean()) if uf.any() else 0.0,
                 max_rel_depth_unflagged=float(rel[uf].max()) if uf.any() else 0.0,
                 p9999_rel_depth=float(np.quantile(rel[uf], 0.9999)) if uf.any() else 0.0,
                 max_abs_flagged_vs_nominal=float(err_abs[fl].max()) if fl.any() else 0.0)
    abs_ch, rel_ch, _ = _channels(cam)
    names = ["r", "g", "b", "depth", "nx", "ny", "nz", "alpha"] if cam else ["range", "intensity", "raydrop", "alpha"]
    stats["per_channel_unflagged"] = {
        names[c]: dict(max=float(np.abs(g[uf, c] - r[uf, c]).max()) if uf.any() else 0.0,
                       p9999=float(np.quantile(np.abs(g[uf, c] - r[uf, c]), 0.9999)) if uf.any() else 0.0,
                       mean=float(np.abs(g[uf, c] - r[uf, c]).mean()) if uf.any() else 0.0)
        for c in range(C)}
    stats["ok"] = (stats["bad"] == 0 and stats["bad_flagged"] == 0 and unresolved == 0 and
                   stats["ambiguous"] <= max(2, MAX_AMBIGUOUS_FRAC * len(rays)))
    if stats["bad"] or stats["bad_flagged"]:
        i = np.nonzero(bad | bad_flagged)[0][:5]
        stats["worst"] = [dict(ray=int(rays[k]), x=int(rays[k] % W), y=int(rays[k] // W), flag=int(flags[k]),
                               gpu=g[k].round(7).tolist(), ref=r[k].round(7).tolist()) for k in i]
    return stats


def cpu_bin_sort(rect, key, ntx, ntiles):
    """Reference binning from the GPU's own per-surfel arrays: enumerate each
    visible surfel's tiles row-major (tile column modulo ntx), stable-sort the
    pairs by (tile, depth-key bits, surfel index), extract [start,end) ranges."""
    vis = np.nonzero((rect[:, 2] >= rect[:, 0]) & (rect[:, 3] >= rect[:, 1]))[0]
    if len(vis) == 0:
        return np.zeros(0, np.uint32), np.zeros(0, np.uint64), np.zeros((ntiles, 2), np.uint32)
    # vectorised enumeration: per visible surfel a (w x h) block of tiles
    x0, y0, x1, y1 = (rect[vis, k].astype(np.int64) for k in range(4))
    w, h = x1 - x0 + 1, y1 - y0 + 1
    cnt = w * h
    ids = np.repeat(vis.astype(np.int64), cnt)
    start = np.repeat(np.cumsum(cnt) - cnt, cnt)
    k = np.arange(int(cnt.sum()), dtype=np.int64) - start
    wr = np.repeat(w, cnt)
    ty = np.repeat(y0, cnt) + k // wr
    tx = np.repeat(x0, cnt) + k % wr
    tiles = (ty * ntx + np.where(tx >= ntx, tx - ntx, tx)).astype(np.uint64)
    kk = (tiles << np.uint64(32)) | key[ids].astype(np.uint64)
    order = np.lexsort((ids, kk))
    vals = ids[order].astype(np.uint32)
    keys = kk[order]
    t_sorted = (keys >> np.uint64(32)).astype(np.int64)
    ranges = np.zeros((ntiles, 2), np.uint32)
    starts = np.searchsorted(t_sorted, np.arange(ntiles), side="left")
    ends = np.searchsorted(t_sorted, np.arange(ntiles), side="right")
    nz = ends > starts
    ranges[nz, 0] = starts[nz]
    ranges[nz, 1] = ends[nz]
    return vals, keys, ranges
