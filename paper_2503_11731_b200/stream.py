"""Chunk streaming with double-buffered residency.

PAPER.md:123 (§III-A "Support Large-scale Scenes"): the scene is split by
XOY location into 40 x 40 m zones with 25 % relative padding; "during
rendering, we use two threads for double-buffering, swapping-in related
Gaussians when the vehicle is moving between two blocks".

B200 design: the chunks live in pinned host memory; the GPU
holds two surfel buffers (front, back), each sized for the largest active
set.  `ChunkStreamer.update(position)` computes the pose's active set (every
zone whose padded XOY box -- 1.25x the zone, reading N9 -- contains the ego
position); when it
differs from the front buffer's set, the new set is copied into the back
buffer with asynchronous host->device copies on a dedicated copy stream (the
second "thread" of the paper is this stream: no host thread blocks), and an
event marks completion.  Rendering keeps using the front buffer -- bitwise
the same frames as before the upload began -- and the buffers swap only when
the back buffer is complete (`poll()`), so a render never sees a partially
uploaded set.  A set is the concatenation of its chunks in chunk order,
so surfel order (and depth-tie order, reading R9) is deterministic.

Plumbing only: buffers, copies and events are PyTorch; every rendering step
runs in libgsr.so (Renderer / BatchRenderer render from `front()`).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import gsr, render

FIELDS = ("means", "quats", "scales", "opacities", "sh", "intensity", "raydrop_logit")


@dataclass
class Zone:
    """A chunk's XOY extent (world x and z; y is up) before padding."""
    x0: float
    x1: float
    z0: float
    z1: float

    def padded_contains(self, x: float, z: float, pad: float) -> bool:
        """The zone grown by `pad` of its size in each axis (pad / 2 per side)."""
        px, pz = 0.5 * pad * (self.x1 - self.x0), 0.5 * pad * (self.z1 - self.z0)
        return (self.x0 - px <= x <= self.x1 + px) and (self.z0 - pz <= z <= self.z1 + pz)


def active_set(zones, position, pad: float = 0.25):
    """Chunk ids whose zone, grown by the relative padding `pad` (the padded
    zone is (1 + pad) times the zone in each axis, reading N9), contains the
    ego's XOY position (world x, z), in chunk order."""
    x, z = float(position[0]), float(position[2])
    return tuple(i for i, zn in enumerate(zones) if zn.padded_contains(x, z, pad))


class ChunkStreamer:
    def __init__(self, chunks, zones, device="cuda", pad: float = 0.25, max_active: int | None = None):
        """chunks: list of scenegen.Surfels (one per zone, same attribute set);
        zones: their XOY extents.  The device buffers hold the largest active
        set over the zone centres and boundaries (or `max_active` chunks)."""
        assert len(chunks) == len(zones) and chunks
        self.device = torch.device(device)
        self.zones, self.pad = list(zones), float(pad)
        self.sh_degree = int(chunks[0].sh_degree)
        self.counts = [c.n for c in chunks]
        # pinned host copies of every chunk (the scene's home when it exceeds HBM)
        self.host = []
        for c in chunks:
            h = {}
            for f in FIELDS:
                a = getattr(c, f)
                h[f] = None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).pin_memory()
            self.host.append(h)
        if max_active is None:
            cap = 0
            for zn in self.zones:
                for x in (zn.x0, 0.5 * (zn.x0 + zn.x1), zn.x1):
                    for z in (zn.z0, 0.5 * (zn.z0 + zn.z1), zn.z1):
                        cap = max(cap, sum(self.counts[i] for i in active_set(self.zones, (x, 0.0, z), pad)))
        else:
            cap = sum(sorted(self.counts)[-max_active:])
        self.capacity = int(cap)
        self.buf = [self._alloc(self.capacity), self._alloc(self.capacity)]
        self.sets = [None, None]          # chunk ids held by buffer 0 / 1
        self.front_i = 0
        self.pending = None               # (buffer index, ids, event) of an upload in flight
        self.copy_stream = torch.cuda.Stream(self.device)
        self.bytes_uploaded = 0
        self.swaps = 0

    def _alloc(self, n):
        h = self.host[0]
        b = {f: (None if h[f] is None else torch.empty((n,) + tuple(h[f].shape[1:]), dtype=torch.float32,
                                                       device=self.device)) for f in FIELDS}
        b["cull_bounds"] = torch.empty((max(gsr.gs_cull_blocks(n), 1), 8), dtype=torch.float32, device=self.device)
        return b

    def _view(self, i):
        ids = self.sets[i]
        n = sum(self.counts[c] for c in ids) if ids is not None else 0
        d = {f: (None if t is None else t[:n]) for f, t in self.buf[i].items() if f != "cull_bounds"}
        d["sh_degree"] = self.sh_degree
        d["cull_bounds"] = self.buf[i]["cull_bounds"]   # of the first n surfels (computed by _upload)
        return d

    def front(self) -> dict:
        """The surfel set renders use now (render.to_device format)."""
        return self._view(self.front_i)

    def front_set(self):
        return self.sets[self.front_i]

    def _upload(self, i, ids):
        """Copy chunks `ids` into buffer i on the copy stream; returns the completion event."""
        n = sum(self.counts[c] for c in ids)
        if n > self.capacity:
            raise RuntimeError(f"active set of {n} surfels exceeds the buffer capacity {self.capacity}")
        # the previous renders from buffer i (issued on the current stream) must finish first
        self.copy_stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.copy_stream):
            off = 0
            for c in ids:
                k = self.counts[c]
                for f in FIELDS:
                    src = self.host[c][f]
                    if src is not None:
                        self.buf[i][f][off:off + k].copy_(src, non_blocking=True)
                        self.bytes_uploaded += src.numel() * 4
                off += k
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.sets[i] = None               # incomplete until the event
        return ev

    def load(self, position):
        """Synchronously make the pose's active set the front buffer (start-up)."""
        ids = active_set(self.zones, position, self.pad)
        ev = self._upload(self.front_i, ids)
        ev.synchronize()
        self.sets[self.front_i] = ids
        self._bounds(self.front_i)
        return ids

    def _bounds(self, i):
        """Block bounds of buffer i's set (hierarchical cull, gs_cull_bounds), on the
        current stream once the upload is complete: a kernel queued behind the copy
        stream's transfers would hold up other streams sharing its hardware queue."""
        n = sum(self.counts[c] for c in self.sets[i])
        render.cull_bounds(dict(self.buf[i], sh_degree=self.sh_degree), n=n)

    def update(self, position) -> bool:
        """Start uploading the pose's active set into the back buffer if it
        differs from the front (and from an upload already in flight).
        Returns True if an upload was started."""
        ids = active_set(self.zones, position, self.pad)
        if ids == self.sets[self.front_i] or (self.pending is not None and self.pending[1] == ids):
            return False
        if self.pending is not None:      # superseded: let it finish, then reuse the buffer
            self.pending[2].synchronize()
        back = 1 - self.front_i
        ev = self._upload(back, ids)
        self.pending = (back, ids, ev)
        return True

    def poll(self, wait: bool = False) -> bool:
        """Swap front and back if the back buffer's upload is complete (or
        wait for it).  Returns True if a swap happened.  Renders enqueued
        after a swap read the new set; the current stream is ordered after
        the upload."""
        if self.pending is None:
            return False
        back, ids, ev = self.pending
        if not (wait or ev.query()):
            return False
        torch.cuda.current_stream(self.device).wait_event(ev)
        self.sets[back] = ids
        self._bounds(back)
        self.front_i = back
        self.pending = None
        self.swaps += 1
        return True


def chunked_zones(n_chunks: int = 8, length: float = 50.0, half_width: float = 10.0):
    """The Chunked street's zones: chunk c covers z in [50c, 50c + 50) and the
    street's lateral extent (scenegen.chunked_surfels)."""
    return [Zone(-half_width, half_width, length * c, length * (c + 1)) for c in range(n_chunks)]
