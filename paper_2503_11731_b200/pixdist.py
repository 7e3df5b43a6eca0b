"""Pixel-partitioned rendering of ONE frame over several GPUs (SURVEY.md
§8(f) NEXT-4; §III-A "Paralleled training").

The paper's training-time multi-GPU scheme, adapted to forward rendering of
a frame too large for one GPU's time budget:

  (1) "an adaptive strategy based on rendering time to allocate continuous
      image regions across multiple GPUs": the image is split into bands of
      tile rows, one per rank; `adapt_bands` moves the boundaries so every
      band gets the same predicted time, predicting each tile row's time from
      its pair count and the time per pair its band measured last frame;
  (2) the surfels are distributed: rank r owns a contiguous shard of the
      global surfel array;
  (3) "a sparse all-to-all communication scheme to transfer the required
      Gaussian data to corresponding pixel partitions": each rank projects
      its shard (gs_project), routes every visible surfel to the bands its
      tile rect overlaps (gs_band_route), packs those surfels' attributes per
      destination (gs_pack_surfels) and one all_to_all_single (NCCL) moves
      only them.  The receiver unpacks the payloads in source-rank order --
      global surfel order, so depth ties keep the single-GPU order (reading
      R9) -- and renders its band through the band's cropped sensor (same
      rays: c_y shifted by the band's first row; LiDAR: its beams).

Unsplit tile lists give band images bitwise equal to the single-GPU frame
(tests/test_gpu_pixdist.py).  Host logic only (buffers, band tables, the
collective): the projection, routing, packing and rendering run in
libgsr.so.  `emulate` runs the same steps for all ranks in one process (one
GPU, ranks one after another, no inter-rank waits).
"""
from __future__ import annotations

import copy

import numpy as np
import torch

from . import gsr
from .render import Renderer, n_channels


# ---------------------------------------------------------------- band tables (host)
def tile_rows(sensor, opts: gsr.gs_opts) -> int:
    return (int(sensor.height) + int(opts.tile_h) - 1) // int(opts.tile_h)


def balanced_bands(cost_rows, n_bands: int):
    """Boundaries [0 = b_0 < b_1 < ... < b_nb = rows] of n_bands contiguous
    bands of tile rows with (greedily) equal summed cost; every band gets at
    least one row."""
    cost = np.maximum(np.asarray(cost_rows, np.float64), 0.0)
    rows = len(cost)
    n_bands = max(1, min(int(n_bands), rows))
    if cost.sum() <= 0:
        cost = np.ones(rows)
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [0]
    for b in range(1, n_bands):
        target = cum[-1] * b / n_bands
        r = int(np.searchsorted(cum, target, side="left"))
        # the row boundary closest to the target, keeping >= 1 row per band
        if r > 0 and abs(cum[r - 1] - target) <= abs(cum[min(r, rows)] - target):
            r -= 1
        r = max(r, bounds[-1] + 1)
        r = min(r, rows - (n_bands - b))
        bounds.append(r)
    bounds.append(rows)
    return bounds


def adapt_bands(bounds, band_ms, row_pairs):
    """Time-adaptive re-partition: predicted time of tile row r in band b =
    row_pairs[r] * band_ms[b] / (pairs of band b) (rows of a band without
    pairs share its time evenly); new bounds balance the predicted times."""
    row_pairs = np.asarray(row_pairs, np.float64)
    cost = np.zeros(len(row_pairs))
    for b in range(len(bounds) - 1):
        lo, hi = bounds[b], bounds[b + 1]
        tot = row_pairs[lo:hi].sum()
        cost[lo:hi] = (row_pairs[lo:hi] * band_ms[b] / tot) if tot > 0 else band_ms[b] / (hi - lo)
    return balanced_bands(cost, len(bounds) - 1)


def band_sensor(sensor, row0: int, row1: int):
    """The sensor restricted to pixel rows [row0, row1): the same rays for
    those rows (cameras: c_y - row0; LiDAR: beams row0..row1-1)."""
    s = copy.copy(sensor)
    s.height = int(row1 - row0)
    if int(sensor.kind) == gsr.GS_LIDAR_SPINNING:
        s.beam_elevation = np.ascontiguousarray(np.asarray(sensor.beam_elevation, np.float32)[row0:row1])
    else:
        s.cy = float(np.float32(np.float64(sensor.cy) - row0))
        assert np.float64(s.cy) + row0 == np.float64(sensor.cy), "c_y - row0 must be exact in fp32"
    return s


def shard_surfels(surfels: dict, world: int, rank: int) -> dict:
    """Rank's contiguous shard of a device surfel dict (views, no copy)."""
    n = int(surfels["means"].shape[0])
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    # the whole set's block bounds do not describe a shard: the shard renders without
    # (render.cull_bounds(shard) would give it its own)
    return {k: (v[lo:hi] if isinstance(v, torch.Tensor) else v) for k, v in surfels.items() if k != "cull_bounds"}


# ---------------------------------------------------------------- per-rank steps (device)
class BandRouter:
    """Project a surfel shard for a frame, route it to bands and pack the
    per-band payloads (one rank's send side)."""

    def __init__(self, shard: dict, opts: gsr.gs_opts | None = None, device="cuda"):
        self.r = Renderer(shard, opts, device)
        self.t = shard
        self.device = self.r.device

    def route(self, sensor, bounds, stream=None):
        """-> (payload [sum counts, F] ordered by band, counts [nb] (host ints))."""
        if not isinstance(sensor, gsr.Sensor):
            sensor = gsr.Sensor(sensor)
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        proj, _ = self.r.project(sensor, st)
        n, nb = self.r.n, len(bounds) - 1
        counts = torch.empty(nb, dtype=torch.int32, device=self.device)
        index = self.r._i32("route_index", max(1, nb * n))
        ws = self.r._get("route_ws", gsr.gs_band_route_workspace_bytes(n, nb))
        gsr.gs_band_route(proj, n, sensor, self.r.opts, bounds, counts, index, ws, st)
        c = [int(x) for x in counts.cpu().tolist()]   # sizes for the all-to-all (one sync)
        sh = self.t.get("sh")
        F = gsr.gs_payload_floats(self.t["sh_degree"] if sh is not None else -1,
                                  self.t.get("intensity") is not None, self.t.get("raydrop_logit") is not None)
        payload = torch.empty((sum(c), F), dtype=torch.float32, device=self.device)
        src = gsr.surfels_struct(self.t)
        off = 0
        for b in range(nb):
            if c[b]:
                gsr.gs_pack_surfels(src, index[b * n: b * n + c[b]], c[b], payload[off: off + c[b]], st)
            off += c[b]
        return payload, c


def unpack(payload: torch.Tensor, like: dict) -> dict:
    """Received payload rows -> a device surfel dict with `like`'s attribute set."""
    m = int(payload.shape[0])
    dev = payload.device
    f = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)
    sh = like.get("sh")
    deg = like["sh_degree"] if sh is not None else -1
    out = dict(means=f(m, 3), quats=f(m, 4), scales=f(m, 2), opacities=f(m),
               sh=f(m, (deg + 1) ** 2, 3) if sh is not None else None, sh_degree=like["sh_degree"],
               intensity=f(m) if like.get("intensity") is not None else None,
               raydrop_logit=f(m) if like.get("raydrop_logit") is not None else None)
    st = torch.cuda.current_stream(dev).cuda_stream
    gsr.gs_unpack_surfels(payload, m, deg, out["intensity"] is not None, out["raydrop_logit"] is not None,
                          out["means"], out["quats"], out["scales"], out["opacities"], out["sh"],
                          out["intensity"], out["raydrop_logit"], st)
    return out


def exchange(payload: torch.Tensor, counts, group=None):
    """Sparse all-to-all of variable-size payload rows: rank r sends rows
    [sum(counts[:d]), sum(counts[:d+1])) to rank d; returns the received rows
    in source-rank order and the per-source counts."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = payload.device
    send_c = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv_c = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_c, send_c, group=group)
    rc = [int(x) for x in recv_c.cpu().tolist()]
    F = payload.shape[1]
    recv = torch.empty((sum(rc), F), dtype=payload.dtype, device=dev)
    dist.all_to_all_single(recv, payload.contiguous(), output_split_sizes=rc, input_split_sizes=list(counts),
                           group=group)
    return recv, rc


class PixelPartitionRenderer:
    """One rank of the pixel-partitioned frame render (torch.distributed)."""

    def __init__(self, surfels: dict, world: int, rank: int, opts: gsr.gs_opts | None = None, group=None,
                 device="cuda"):
        self.world, self.rank, self.group = world, rank, group
        self.shard = shard_surfels(surfels, world, rank)
        self.opts = opts if opts is not None else gsr.default_opts()
        self.router = BandRouter(self.shard, self.opts, device)
        self.device = self.router.device

    def render(self, sensor, bounds):
        """Render this rank's band of `sensor` (tile-row bounds, one band per
        rank).  Returns (band image [C, rows, W], stats)."""
        payload, counts = self.router.route(sensor, bounds)
        recv, rc = exchange(payload, counts, self.group)
        band = unpack(recv, self.shard)
        th = int(self.opts.tile_h)
        r0, r1 = bounds[self.rank] * th, min(bounds[self.rank + 1] * th, int(sensor.height))
        img = Renderer(band, self.opts, self.device).render(band_sensor(sensor, r0, r1))
        return img, {"sent": sum(counts), "received": sum(rc), "per_source": rc}


def emulate(surfels: dict, sensor, bounds, world: int, opts: gsr.gs_opts | None = None, device="cuda"):
    """All ranks' steps in one process, one after another (one GPU): project
    + route + pack every shard, then assemble each band's payload in
    source-rank order, unpack and render it.  Returns (full frame [C,H,W],
    per-band surfel counts, per-(source, band) counts)."""
    opts = opts if opts is not None else gsr.default_opts()
    nb = len(bounds) - 1
    sends = []
    for r in range(world):
        sh = shard_surfels(surfels, world, r)
        payload, counts = BandRouter(sh, opts, device).route(sensor, bounds)
        sends.append((payload, counts))
    th = int(opts.tile_h)
    C = n_channels(int(sensor.kind))
    full = torch.empty((C, int(sensor.height), int(sensor.width)), dtype=torch.float32, device=device)
    band_n, matrix = [], []
    for b in range(nb):
        parts = []
        for payload, counts in sends:
            off = sum(counts[:b])
            parts.append(payload[off: off + counts[b]])
        matrix.append([c[b] for _, c in sends])
        recv = torch.cat(parts, 0) if parts else None
        band = unpack(recv, surfels)
        band_n.append(int(recv.shape[0]))
        r0, r1 = bounds[b] * th, min(bounds[b + 1] * th, int(sensor.height))
        full[:, r0:r1] = Renderer(band, opts, device).render(band_sensor(sensor, r0, r1))
    return full, band_n, matrix
