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


def check_sorted_pairs(b, ntx):
    """The GPU's sorted pair list is a valid binning of the tile set it
    emitted: (tile, depth-key bits, surfel index) strictly increasing, each
    pair's key bits = its surfel's key, every visible surfel emitted exactly
    count[i] distinct pairs inside its rect, and the tile ranges are the
    [start, end) runs of the sorted tiles (bit-exact).  Returns the pairs'
    (tile, surfel) arrays for further checks."""
    P = b["P"]
    vals = b["values"].astype(np.int64)
    keys = b["keys"]
    assert len(vals) == P and len(keys) == P
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    kb = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    np.testing.assert_array_equal(kb, b["key"][vals])
    if P > 1:
        t0, t1 = tiles[:-1], tiles[1:]
        k0, k1 = kb[:-1], kb[1:]
        v0, v1 = vals[:-1], vals[1:]
        inc = (t0 < t1) | ((t0 == t1) & ((k0 < k1) | ((k0 == k1) & (v0 < v1))))
        assert inc.all(), f"sorted pairs out of order at {np.nonzero(~inc)[0][:5]}"
    n = len(b["count"])
    cnt = np.bincount(vals, minlength=n)
    np.testing.assert_array_equal(cnt, b["count"].astype(np.int64))
    rect = b["rect"].astype(np.int64)
    tx = tiles % ntx
    ty = tiles // ntx
    tx = np.where(tx < rect[vals, 0], tx + ntx, tx)   # LiDAR rects may run past the seam (columns >= ntx)
    inside = (tx >= rect[vals, 0]) & (tx <= rect[vals, 2]) & (ty >= rect[vals, 1]) & (ty <= rect[vals, 3])
    assert inside.all(), f"{int((~inside).sum())} pairs outside their surfel's rect"
    if len(vals):   # each (tile, surfel) pair once
        u = np.unique(tiles * (1 << 32) + vals)
        assert len(u) == len(vals), "duplicate (tile, surfel) pairs"
    ranges = np.zeros((b["ntiles"], 2), np.uint32)
    starts = np.searchsorted(tiles, np.arange(b["ntiles"]), side="left")
    ends = np.searchsorted(tiles, np.arange(b["ntiles"]), side="right")
    nz = ends > starts
    ranges[nz, 0] = starts[nz]
    ranges[nz, 1] = ends[nz]
    np.testing.assert_array_equal(b["ranges"], ranges)
    return tiles, vals


def required_pinhole_pairs(surfels, sensor, tile_w, tile_h, idx=None, near=0.2, support=9.0, sigma=0.70710678,
                           alpha_min=1.0 / 255.0, margin=1e-4, max_window=1 << 16):
    """(tile, surfel) pairs a pinhole binning must contain, from an fp64
    evaluation of the definition (Eq. 2 intersection of the
    pixel-centre ray with the surfel plane, the 3-sigma cut rho <= support
    with the opacity-aware alpha cut, the low-pass floor, the near plane),
    independent of the GPU records: every tile holding a pixel centre where
    the surfel contributes with a relative margin `margin` inside every cut.
    Pixel centres are enumerated over the projected 3-sigma circle's box
    (256 boundary points) and the low-pass disc, widened by 2 px; surfels
    whose boundary crosses the near plane or whose window exceeds
    max_window pixels are skipped (returned count)."""
    W, H = sensor.width, sensor.height
    Wm = np.asarray(sensor.world_to_sensor, np.float64)
    Rs, ts = Wm[:, :3], Wm[:, 3]
    n = surfels.n
    idx = np.arange(n) if idx is None else np.asarray(idx)
    mu = surfels.means[idx].astype(np.float64) @ Rs.T + ts
    q = surfels.quats[idx].astype(np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    tu = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], 1) @ Rs.T
    tv = np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], 1) @ Rs.T
    a = tu * surfels.scales[idx, 0:1].astype(np.float64)
    bb = tv * surfels.scales[idx, 1:2].astype(np.float64)
    o = surfels.opacities[idx].astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        rcut = np.minimum(support, 2.0 * np.log(o / alpha_min))
    fx, fy, cx, cy = float(sensor.fx), float(sensor.fy), float(sensor.cx), float(sensor.cy)
    ok = (mu[:, 2] > near) & (rcut > 0) & np.isfinite(rcut)
    ang = np.linspace(0, 2 * np.pi, 256, endpoint=False)
    R3 = np.sqrt(np.maximum(rcut, 0))
    pts = mu[:, None, :] + R3[:, None, None] * (np.cos(ang)[None, :, None] * a[:, None, :] +
                                                np.sin(ang)[None, :, None] * bb[:, None, :])
    front = (pts[:, :, 2] > near).all(axis=1)
    px = fx * pts[:, :, 0] / np.where(front[:, None], pts[:, :, 2], 1.0) + cx
    py = fy * pts[:, :, 1] / np.where(front[:, None], pts[:, :, 2], 1.0) + cy
    ccx = fx * mu[:, 0] / mu[:, 2] + cx
    ccy = fy * mu[:, 1] / mu[:, 2] + cy
    rlp = sigma * R3
    x0 = np.floor(np.minimum(px.min(1), ccx - rlp) - 2).clip(0, W - 1).astype(np.int64)
    x1 = np.ceil(np.maximum(px.max(1), ccx + rlp) + 2).clip(0, W - 1).astype(np.int64)
    y0 = np.floor(np.minimum(py.min(1), ccy - rlp) - 2).clip(0, H - 1).astype(np.int64)
    y1 = np.ceil(np.maximum(py.max(1), ccy + rlp) + 2).clip(0, H - 1).astype(np.int64)
    win = (x1 - x0 + 1) * (y1 - y0 + 1)
    use = ok & front & (win <= max_window)
    skipped = int(np.sum(ok & ~use))
    out = []
    sel = np.nonzero(use)[0]
    for chunk in np.array_split(sel, max(1, int(win[sel].sum() // 4_000_000) + 1)):
        if len(chunk) == 0:
            continue
        cw = win[chunk]
        rep = np.repeat(chunk, cw)
        k = np.arange(int(cw.sum())) - np.repeat(np.cumsum(cw) - cw, cw)
        ww = (x1 - x0 + 1)[rep]
        pxi = x0[rep] + k % ww
        pyi = y0[rep] + k // ww
        dx = (pxi + 0.5 - cx) / fx
        dy = (pyi + 0.5 - cy) / fy
        d = np.stack([dx, dy, np.ones_like(dx)], 1)
        A, B, M = a[rep], bb[rep], mu[rep]
        # mu + u a + v b = lam d  ->  [a b -d][u v lam]^T = -mu (Cramer)
        Dm = -d
        det = np.einsum("ij,ij->i", A, np.cross(B, Dm))
        rhs = -M
        with np.errstate(divide="ignore", invalid="ignore"):
            u = np.einsum("ij,ij->i", rhs, np.cross(B, Dm)) / det
            v = np.einsum("ij,ij->i", A, np.cross(rhs, Dm)) / det
            lam = np.einsum("ij,ij->i", A, np.cross(B, rhs)) / det
        rho3 = u * u + v * v
        rho2 = ((pxi + 0.5 - ccx[rep]) ** 2 + (pyi + 0.5 - ccy[rep]) ** 2) / (sigma * sigma)
        use3 = rho3 <= rho2
        rho = np.where(use3, rho3, rho2)
        dep = np.where(use3, lam, mu[rep, 2])
        lim = rcut[rep] * (1 - margin)
        need = np.isfinite(rho) & (rho <= lim) & (dep >= near * (1 + margin))
        t = (pyi[need] // tile_h) * ((W + tile_w - 1) // tile_w) + pxi[need] // tile_w
        out.append(np.unique(t.astype(np.int64) * (1 << 32) + idx[rep[need]]))
    pairs = np.unique(np.concatenate(out)) if out else np.zeros(0, np.int64)
    return pairs >> 32, pairs & 0xFFFFFFFF, skipped


def check_pinhole_binning(b, surfels, sensor, tile_w, tile_h, idx=None, **kw):
    """Sorted-pair validity (check_sorted_pairs) plus conservativeness: every
    required (tile, surfel) pair of the fp64 definition is emitted."""
    ntx = (sensor.width + tile_w - 1) // tile_w
    tiles, vals = check_sorted_pairs(b, ntx)
    rt, rs, skipped = required_pinhole_pairs(surfels, sensor, tile_w, tile_h, idx=idx, **kw)
    have = np.unique(tiles * (1 << 32) + vals)
    need = rt * (1 << 32) + rs
    missing = np.setdiff1d(need, have)
    assert len(missing) == 0, f"{len(missing)} required pairs missing, e.g. tile/surfel " \
                              f"{[(int(m >> 32), int(m & 0xFFFFFFFF)) for m in missing[:5]]}"
    return dict(P=b["P"], required=len(need), skipped=skipped)


def required_lidar_pairs(surfels, sensor, tile_w, idx=None, near=0.2, support=9.0, alpha_min=1.0 / 255.0,
                         margin=1e-4, max_window=1 << 16):
    """(tile, surfel) pairs a LiDAR binning (tile = tile_w columns of one beam
    row) must contain, from an fp64 evaluation of the definition (Eq. 5 rays,
    Eq. 2 intersection, 3-sigma cut with the opacity-aware alpha cut, near
    plane; no low-pass, reading R6): every tile holding a ray that meets the
    surfel with a relative margin inside every cut.  Rays are enumerated over
    the angular window of the 3-sigma circle (256 boundary points), widened by
    two beams / columns; surfels whose window wraps the whole turn or exceeds
    max_window rays are skipped (returned count)."""
    W, H = sensor.width, sensor.height
    ntx = (W + tile_w - 1) // tile_w
    Wm = np.asarray(sensor.world_to_sensor, np.float64)
    Rs, ts = Wm[:, :3], Wm[:, 3]
    idx = np.arange(surfels.n) if idx is None else np.asarray(idx)
    mu = surfels.means[idx].astype(np.float64) @ Rs.T + ts
    q = surfels.quats[idx].astype(np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    tu = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], 1) @ Rs.T
    tv = np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], 1) @ Rs.T
    a = tu * surfels.scales[idx, 0:1].astype(np.float64)
    bb = tv * surfels.scales[idx, 1:2].astype(np.float64)
    o = surfels.opacities[idx].astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        rcut = np.minimum(support, 2.0 * np.log(o / alpha_min))
    ok = (np.linalg.norm(mu, axis=1) > near) & (rcut > 0) & np.isfinite(rcut)
    R3 = np.sqrt(np.maximum(rcut, 0))
    ang = np.linspace(0, 2 * np.pi, 256, endpoint=False)
    pts = mu[:, None, :] + R3[:, None, None] * (np.cos(ang)[None, :, None] * a[:, None, :] +
                                                np.sin(ang)[None, :, None] * bb[:, None, :])
    el = np.arctan2(pts[:, :, 2], np.hypot(pts[:, :, 0], pts[:, :, 1]))
    azc = np.arctan2(mu[:, 1], mu[:, 0])
    daz = np.angle(np.exp(1j * (np.arctan2(pts[:, :, 1], pts[:, :, 0]) - azc[:, None])))
    beams = np.asarray(sensor.beam_elevation, np.float64)
    bstep = np.abs(np.diff(beams)).max() if H > 1 else 1.0
    az0, step = float(sensor.azimuth0), float(sensor.azimuth_step)
    # the sensor origin inside the disk's cone (all azimuths): skip
    wide = (daz.max(1) - daz.min(1)) > np.pi
    j0 = np.floor((azc + daz.min(1) - az0) / step).astype(np.int64) - 2
    j1 = np.ceil((azc + daz.max(1) - az0) / step).astype(np.int64) + 2
    lo_el, hi_el = el.min(1) - 2 * bstep, el.max(1) + 2 * bstep
    rows = [np.nonzero((beams >= lo_el[k]) & (beams <= hi_el[k]))[0] for k in range(len(idx))]
    ncol = np.minimum(j1 - j0 + 1, W)
    nrow = np.array([len(r) for r in rows])
    use = ok & ~wide & (ncol * nrow <= max_window) & (nrow > 0)
    skipped = int(np.sum(ok & ~use))
    out = []
    for k in np.nonzero(use)[0]:
        rr = rows[k]
        jj = j0[k] + np.arange(ncol[k])
        th = beams[rr][:, None]
        ph = az0 + np.mod(jj, W)[None, :] * step
        d = np.stack(np.broadcast_arrays(np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), np.sin(th)), -1).reshape(-1, 3)
        A, B, M = a[k], bb[k], mu[k]
        Dm = -d
        det = (np.cross(B, Dm) @ A)
        with np.errstate(divide="ignore", invalid="ignore"):
            u = (np.cross(B, Dm) @ (-M)) / det
            v = np.einsum("j,ij->i", A, np.cross(-M[None, :], Dm)) / det
            lam = np.einsum("j,ij->i", A, np.cross(B[None, :], -M[None, :])) / det
        rho = u * u + v * v
        need = np.isfinite(rho) & (rho <= rcut[k] * (1 - margin)) & (lam >= near * (1 + margin))
        r_idx = np.repeat(rr, len(jj))[need]
        c_idx = np.tile(np.mod(jj, W), len(rr))[need]
        t = r_idx * ntx + c_idx // tile_w
        out.append(np.unique(t.astype(np.int64) * (1 << 32) + idx[k]))
    pairs = np.unique(np.concatenate(out)) if out else np.zeros(0, np.int64)
    return pairs >> 32, pairs & 0xFFFFFFFF, skipped


def check_lidar_binning(b, surfels, sensor, tile_w, idx=None, **kw):
    """Sorted-pair validity plus conservativeness (required_lidar_pairs)."""
    ntx = (sensor.width + tile_w - 1) // tile_w
    tiles, vals = check_sorted_pairs(b, ntx)
    rt, rs, skipped = required_lidar_pairs(surfels, sensor, tile_w, idx=idx, **kw)
    have = np.unique(tiles * (1 << 32) + vals)
    need = rt * (1 << 32) + rs
    missing = np.setdiff1d(need, have)
    assert len(missing) == 0, f"{len(missing)} required pairs missing, e.g. tile/surfel " \
                              f"{[(int(m >> 32), int(m & 0xFFFFFFFF)) for m in missing[:5]]}"
    return dict(P=b["P"], required=len(need), skipped=skipped)
