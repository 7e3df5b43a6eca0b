"""Frame rendering through the C-ABI (buffer management + the four calls).

`Renderer` keeps a surfel set resident on one GPU and renders sensor frames
with gs_project -> gs_bin_sort -> gs_render_camera / gs_render_lidar.  It only
allocates torch buffers and marshals arguments: every step of the path runs
in libgsr.so.  Two sizing modes (include/gsr.h):

  * exact (default): after gs_project it reads the pair count P (one device
    sync) and sizes the pair buffers to P;
  * capacity: a fixed pair capacity, no host sync (CUDA-graph capturable);
    if the overflow flag is raised the frame is re-rendered with a larger
    capacity (check with `overflowed()`).
"""
from __future__ import annotations

import numpy as np
import torch

from . import gsr

CAMERA_CHANNELS = ("r", "g", "b", "depth", "nx", "ny", "nz", "alpha")
LIDAR_CHANNELS = ("range", "intensity", "raydrop", "alpha")


def to_device(s, device="cuda", bounds: bool = True) -> dict:
    """scenegen.Surfels (numpy fp32) -> dict of contiguous CUDA tensors
    (+ the block bounds of the hierarchical cull, gs_cull_bounds, unless
    bounds=False)."""
    f = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)
    d = dict(means=f(s.means), quats=f(s.quats), scales=f(s.scales), opacities=f(s.opacities),
             sh=f(s.sh), sh_degree=int(s.sh_degree), intensity=f(s.intensity),
             raydrop_logit=f(s.raydrop_logit))
    if bounds:
        cull_bounds(d)
    return d


def cull_bounds(surfels: dict, stream=None, n: int | None = None) -> torch.Tensor:
    """Compute (gs_cull_bounds, on `stream`: a raw CUDA stream handle, default
    the current stream) the block bounds of the first n surfels (default all)
    of a to_device dict into surfels["cull_bounds"] (allocated on first use,
    sized for the whole buffers).  Call again whenever means or scales change."""
    means = surfels["means"]
    b = surfels.get("cull_bounds")
    if b is None:
        b = torch.empty((max(gsr.gs_cull_blocks(means.shape[0]), 1), 8), dtype=torch.float32, device=means.device)
        surfels["cull_bounds"] = b
    st = stream if stream is not None else torch.cuda.current_stream(means.device).cuda_stream
    view = {k: (v[: n] if (n is not None and isinstance(v, torch.Tensor) and k != "cull_bounds") else v)
            for k, v in surfels.items() if k != "cull_bounds"}
    gsr.gs_cull_bounds(gsr.surfels_struct(view), b, st)
    return b


def n_channels(kind):
    return 4 if kind == gsr.GS_LIDAR_SPINNING else 8


class Renderer:
    def __init__(self, surfels: dict, opts: gsr.gs_opts | None = None, device="cuda",
                 lidar_tile=(32, 1)):
        """opts apply to every frame; LiDAR frames use `lidar_tile` (columns x
        beams of one binning tile) unless it is None."""
        self.device = torch.device(device)
        self.t = surfels
        self.n = int(surfels["means"].shape[0])
        self.struct = gsr.surfels_struct(surfels)
        self.cam_opts = opts if opts is not None else gsr.default_opts()
        self.lidar_opts = gsr.gs_opts.from_buffer_copy(self.cam_opts)
        if lidar_tile is not None:
            self.lidar_opts.tile_w, self.lidar_opts.tile_h = int(lidar_tile[0]), int(lidar_tile[1])
        self.opts = self.cam_opts
        self._buf = {}
        self.last_pairs = None

    def set_surfels(self, surfels: dict):
        """Point the renderer at another device surfel set (e.g. the other
        half of a double buffer, or a streamed active set of another size;
        the work buffers grow on demand)."""
        self.t = surfels
        self.n = int(surfels["means"].shape[0])
        self.struct = gsr.surfels_struct(surfels)

    # buffers are cached per (name) and grown on demand
    def _get(self, name, nbytes):
        b = self._buf.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)
            self._buf[name] = b
        return b

    def _i32(self, name, count):
        return self._get(name, 4 * max(count, 1))[: 4 * max(count, 1)].view(torch.int32)

    def opts_for(self, sensor) -> gsr.gs_opts:
        return self.lidar_opts if sensor.kind == gsr.GS_LIDAR_SPINNING else self.cam_opts

    def project(self, sensor: gsr.Sensor, stream=None, opts: gsr.gs_opts | None = None):
        self.opts = opts if opts is not None else self.opts_for(sensor)
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        proj = self._get("proj", gsr.gs_projected_bytes(self.n, sensor.kind))
        d_np = self._get("np", 8)[:8].view(torch.int64)
        gsr.gs_project(self.struct, sensor, self.opts, proj, d_np, st)
        return proj, d_np

    def render(self, sensor, out: torch.Tensor | None = None, capacity: int | None = None,
               keys: bool = False, stream=None, stats: torch.Tensor | None = None,
               events=None, overflow: torch.Tensor | None = None,
               opts: gsr.gs_opts | None = None, render_stream=None) -> torch.Tensor:
        """Render one frame; returns a planar fp32 tensor [C,H,W] (C = 8 for
        cameras: r,g,b,depth,nx,ny,nz,alpha; 4 for LiDAR: range, intensity,
        raydrop, alpha).  stats: optional int32 [2,H,W] (composited, evaluated
        pairs per sample).  events: optional 4 CUDA events recorded before
        gs_project, gs_bin_sort, the render call and after it.  overflow:
        optional int32 device slot for gs_bin_sort's overflow flag (default:
        a buffer owned by the renderer).  opts: this frame's options instead
        of the renderer's (e.g. another tile shape).  render_stream: a torch
        stream the render call runs on after gs_bin_sort (event-ordered), e.g. one
        of another priority; default: the current stream."""
        if not isinstance(sensor, gsr.Sensor):
            sensor = gsr.Sensor(sensor)
        self.opts = self.opts_for(sensor)
        torch_stream = torch.cuda.current_stream(self.device)
        st = stream if stream is not None else torch_stream.cuda_stream
        if events is not None:
            events[0].record(torch_stream)
        proj, d_np = self.project(sensor, st, opts)
        if events is not None:
            events[1].record(torch_stream)
        if capacity is None:
            cap = int(d_np.item())   # exact sizing (one sync)
        else:
            cap = int(capacity)
        self.last_pairs = cap
        nt = gsr.gs_num_tiles(sensor, self.opts)
        values = self._i32("values", cap)
        ranges = self._i32("ranges", 2 * nt)
        ovf = overflow if overflow is not None else self._i32("overflow", 1)
        ws = self._get("ws", gsr.gs_sort_workspace_bytes(self.n, cap, sensor, self.opts))
        kbuf = self._get("keys", 8 * max(cap, 1))[: 8 * max(cap, 1)].view(torch.int64) if keys else None
        gsr.gs_bin_sort(proj, self.n, sensor, self.opts, kbuf, values, cap, ranges, ws, ovf, st)
        C = n_channels(sensor.kind)
        H, W = sensor.height, sensor.width
        if out is None:
            out = torch.empty((C, H, W), dtype=torch.float32, device=self.device)
        rws = self._get("rws", gsr.gs_render_workspace_bytes(cap, sensor, self.opts))
        if render_stream is not None:
            render_stream.wait_stream(torch_stream)
            torch_stream = render_stream
            st = render_stream.cuda_stream
        if events is not None:
            events[2].record(torch_stream)
        if sensor.kind == gsr.GS_LIDAR_SPINNING:
            gsr.gs_render_lidar(proj, self.n, values, ranges, ovf, sensor, self.opts, rws, out[0],
                                out[1], out[2], out[3], st, stats)
        else:
            gsr.gs_render_camera(proj, self.n, values, ranges, ovf, sensor, self.opts, rws, out[0:3],
                                 out[3], out[4:7], out[7], st, stats)
        if events is not None:
            events[3].record(torch_stream)
        self._last = dict(proj=proj, values=values, ranges=ranges, overflow=ovf, keys=kbuf, cap=cap,
                          ntiles=nt, sensor=sensor)
        return out

    def backward(self, grad_out: torch.Tensor) -> dict:
        """Gradients of sum(grad_out * out) for the last rendered frame w.r.t.
        the surfel attributes (gs_render_backward; pinhole and LiDAR).
        Returns {means, quats, scales, opacities, sh | intensity, raydrop_logit}."""
        L = self._last
        sensor = L["sensor"]
        st = torch.cuda.current_stream(self.device).cuda_stream
        f = lambda t: None if t is None else torch.empty_like(t)
        lidar = sensor.kind == gsr.GS_LIDAR_SPINNING
        g = dict(means=f(self.t["means"]), quats=f(self.t["quats"]), scales=f(self.t["scales"]),
                 opacities=f(self.t["opacities"]), sh=None if lidar else f(self.t.get("sh")),
                 intensity=f(self.t.get("intensity")) if lidar else None,
                 raydrop_logit=f(self.t.get("raydrop_logit")) if lidar else None)
        ws = self._get("bwd_ws", gsr.gs_backward_workspace_bytes(self.n))
        gsr.gs_render_backward(self.struct, sensor, self.opts, L["proj"], L["values"], L["ranges"],
                               grad_out.contiguous(), ws, g["means"], g["quats"], g["scales"], g["opacities"],
                               g["sh"], g["intensity"], g["raydrop_logit"], st)
        return g

    def overflowed(self) -> bool:
        return bool(self._last["overflow"].item())

    def binning_state(self):
        """Host copies of the last frame's per-surfel and sorted-pair arrays
        (for the bit-exact binning test)."""
        L = self._last
        sensor = L["sensor"]
        offs = gsr.gs_projected_offsets(self.n, sensor.kind)
        proj = L["proj"]
        n = self.n
        rect = proj[offs["rect"]: offs["rect"] + 8 * n].view(torch.int16).view(n, 4).cpu().numpy()
        key = proj[offs["key"]: offs["key"] + 4 * n].view(torch.int32).cpu().numpy().view(np.uint32)
        cnt = proj[offs["count"]: offs["count"] + 4 * n].view(torch.int32).cpu().numpy()
        culled = cnt == 0   # rect and key are only defined where the count is > 0 (gsr.h)
        rect = rect.copy()
        rect[culled] = (0, 0, -1, -1)
        key = key.copy()
        key[culled] = 0xFFFFFFFF
        P = int(proj[8:16].view(torch.int64).item())
        vals = L["values"][:P].cpu().numpy().view(np.uint32)
        keys = L["keys"][:P].cpu().numpy().view(np.uint64) if L["keys"] is not None else None
        ranges = L["ranges"][: 2 * L["ntiles"]].cpu().numpy().view(np.uint32).reshape(-1, 2)
        return dict(rect=rect, key=key, count=cnt, P=P, values=vals, keys=keys, ranges=ranges,
                    ntiles=L["ntiles"])
