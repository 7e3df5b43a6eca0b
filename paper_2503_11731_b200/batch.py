"""Batched multi-frame rendering through the C-ABI (many sensor frames over
one resident surfel set), e.g. the Chunked street batch of BASELINE.json
(timesteps x {6 pinholes + 1 LiDAR}).

`BatchRenderer` owns `n_streams` lanes (a `Renderer` buffer set + a CUDA
stream each) and deals frames to them round-robin, so the short serial
kernels of one frame (scans, look-back passes, schedule) overlap the long
ones of the next.  It runs in capacity mode: `plan()` sizes every frame's
pair buffers once (one sync per frame, outside any timed region) and
`render()` is then free of host synchronisation.  Every frame gets its own
overflow slot; `overflowed()` lists frames whose capacity was exceeded.

This module marshals buffers only; all arithmetic runs in libgsr.so.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import gsr
from .render import Renderer, n_channels


@dataclass
class FrameTimes:
    """Per-frame CUDA-event durations (ms) of the three entry points."""
    project: list = field(default_factory=list)
    sort: list = field(default_factory=list)
    render: list = field(default_factory=list)

    @staticmethod
    def from_events(evs) -> "FrameTimes":
        """Durations from recorded (completed) per-frame event quadruples."""
        t = FrameTimes()
        for ev in evs:
            t.project.append(ev[0].elapsed_time(ev[1]))
            t.sort.append(ev[1].elapsed_time(ev[2]))
            t.render.append(ev[2].elapsed_time(ev[3]))
        return t


class BatchRenderer:
    def __init__(self, surfels: dict, opts: gsr.gs_opts | None = None, device="cuda", n_streams: int = 2,
                 lidar_tile=(32, 1), grid_share: float | None = None, big_tile=(16, 16),
                 big_tile_ratio: float = 16.0, priority: str | None = "comp", deal: str = "round_robin",
                 heavy_share: float | None = None):
        """grid_share: fraction of the GPU's resident compositor CTA slots each
        frame's persistent grid takes (gs_opts.grid_share); default 2/n_streams
        (capped at 1), so about two frames composite at once and the other
        streams' projection and binning kernels find free SMs.
        big_tile / big_tile_ratio: plan() bins a camera frame with the larger
        `big_tile` when its surfels cover more than `big_tile_ratio` tiles each
        on average at the default tile (large near surfels: the pair count,
        hence the sort, shrinks ~2x while the compositor hardly slows; the
        Chunked side cameras 1.89 -> 1.72 ms, the forward ones keep 16 x 8).
        None disables it.
        priority: None (one stream per lane) or "pre" / "comp": each lane gets
        a second stream for its render call, and the projection + binning
        stream ("pre") or the compositing stream ("comp") has the higher CUDA
        stream priority (Chunked batch, 10 lanes: none 992, pre 1003, comp
        1010 Msamples/s)."""
        self.device = torch.device(device)
        self.heavy_share = heavy_share   # grid_share of frames with > 1.5x the batch's mean pairs (None: as the others)
        assert deal in ("round_robin", "balanced", "typed"), deal
        self.deal = deal        # how render() deals frames to lanes (see plan())
        self.lane_of = None
        n_streams = max(1, n_streams)
        o = gsr.gs_opts.from_buffer_copy(opts) if opts is not None else gsr.default_opts()
        o.grid_share = float(grid_share) if grid_share is not None else min(1.0, 2.0 / n_streams)
        self.lanes = [Renderer(surfels, o, device, lidar_tile) for _ in range(n_streams)]
        self.big_opts = None
        if big_tile is not None:
            self.big_opts = gsr.gs_opts.from_buffer_copy(o)
            self.big_opts.tile_w, self.big_opts.tile_h = int(big_tile[0]), int(big_tile[1])
        self.big_tile_ratio = float(big_tile_ratio)
        self.frame_opts = None
        self.priority = priority
        if priority is None:
            self.streams = [torch.cuda.Stream(self.device) for _ in self.lanes]
            self.rstreams = [None] * len(self.lanes)
        else:
            assert priority in ("pre", "comp"), priority
            hi, lo = (-1, 0) if priority == "pre" else (0, -1)
            self.streams = [torch.cuda.Stream(self.device, priority=hi) for _ in self.lanes]
            self.rstreams = [torch.cuda.Stream(self.device, priority=lo) for _ in self.lanes]
        self.n = self.lanes[0].n
        self.caps = None
        self.ovf = None

    @staticmethod
    def wrap(sensors):
        return [s if isinstance(s, gsr.Sensor) else gsr.Sensor(s) for s in sensors]

    def alloc_outputs(self, sensors):
        """One planar fp32 output tensor per frame ([8,H,W] camera, [4,H,W] LiDAR)."""
        return [torch.empty((n_channels(s.kind), s.height, s.width), dtype=torch.float32,
                            device=self.device) for s in sensors]

    def plan(self, sensors, stats: bool = False):
        """Exact pair count of every frame -> its capacity (one sync per
        frame).  With stats=True also returns, per frame, the number of
        composited (ray, surfel) pairs and of pairs whose conservative pixel
        box contains the ray (instrumented unsplit kernel)."""
        sensors = self.wrap(sensors)
        lane = self.lanes[0]
        caps, contrib, evals, fopts = [], [], [], []
        for s in sensors:
            proj, d_np = lane.project(s)
            P = int(d_np.item())
            o = None
            if self.big_opts is not None and s.kind != gsr.GS_LIDAR_SPINNING and P > 0:
                V = int(proj[:4].view(torch.int32).item())   # header: visible surfels
                if P > self.big_tile_ratio * V:
                    o = self.big_opts
                    _, d_np = lane.project(s, opts=o)
                    P = int(d_np.item())
            caps.append(P)
            fopts.append(o)
        if self.heavy_share is not None and caps:
            mean = sum(caps) / len(caps)
            for i, P in enumerate(caps):
                if P > 1.5 * mean:
                    o = gsr.gs_opts.from_buffer_copy(fopts[i] if fopts[i] is not None else self.lanes[0].opts_for(sensors[i]))
                    o.grid_share = float(self.heavy_share)
                    fopts[i] = o
        self.caps = caps
        self.frame_opts = fopts
        # deal frames to lanes: round robin (frame i on lane i % lanes), or balanced -- in
        # frame order, each frame to the lane with the least planned work so far (a frame's
        # work ~ 4.3 M pair-equivalents of fixed cost + its pairs: Chunked forward / side /
        # LiDAR frames take 4.0 / 1.4 / 2.4 ms for 27.2 / 6.6 / 11.3 M pairs), so lanes do
        # not specialise on one frame type when the lane count is a multiple of the
        # per-timestep frame count
        if self.deal == "balanced":
            load = [0.0] * len(self.lanes)
            self.lane_of = []
            for P in caps:
                k = min(range(len(load)), key=lambda j: (load[j], j))
                load[k] += 4.3e6 + P
                self.lane_of.append(k)
        elif self.deal == "typed":
            # lanes specialise on a frame class (sensor kind, tile shape, pair count to a
            # power of two) and every class gets lanes in proportion to its planned work;
            # inside a class frames go round robin over the class's lanes
            import math
            cls = [(int(s.kind), fopts[i] is not None, int(round(math.log2(max(P, 1)))))
                   for i, (s, P) in enumerate(zip(sensors, caps))]
            work = {}
            for c, P in zip(cls, caps):
                work[c] = work.get(c, 0.0) + 4.3e6 + P
            L = len(self.lanes)
            keys = sorted(work, key=lambda c: -work[c])[:L]        # more classes than lanes: the lightest share
            tot = sum(work[c] for c in keys)
            share = {c: max(1, int(work[c] / tot * L)) for c in keys}
            while sum(share.values()) > L:
                c = max(share, key=lambda c: (share[c] > 1, share[c] - work[c] / tot * L))
                share[c] -= 1
            while sum(share.values()) < L:
                c = max(share, key=lambda c: work[c] / share[c])
                share[c] += 1
            first, nxt = {}, 0
            for c in keys:
                first[c] = nxt
                nxt += share[c]
            seen = {}
            self.lane_of = []
            for c in cls:
                if c not in first:
                    c = keys[-1]
                j = seen.get(c, 0)
                seen[c] = j + 1
                self.lane_of.append(first[c] + j % share[c])
        else:
            self.lane_of = [i % len(self.lanes) for i in range(len(caps))]
        self.ovf = torch.zeros(len(sensors), dtype=torch.int32, device=self.device)
        if stats:
            for s, cap, o in zip(sensors, caps, fopts):
                st = torch.zeros((2, s.height, s.width), dtype=torch.int32, device=self.device)
                lane.render(s, capacity=cap, stats=st, opts=o)
                tot = st.view(2, -1).sum(dim=1, dtype=torch.int64).cpu()
                contrib.append(int(tot[0]))
                evals.append(int(tot[1]))
        torch.cuda.synchronize(self.device)
        return (caps, contrib, evals) if stats else caps

    def render(self, sensors, outs, times: FrameTimes | None = None, on_frame=None, event_log: list | None = None):
        """Render frame i into outs[i] on lane lane_of[i] (plan()).  times: if given,
        per-frame event durations are appended after the batch completes
        (this synchronises).  event_log: if given, each frame's 4 CUDA events
        (before gs_project, gs_bin_sort, the render call, after it) are
        appended without synchronising (read them after a later sync, e.g.
        with FrameTimes.from_events).  on_frame(i, stream): called right after
        frame i is enqueued (e.g. to chain a device->host copy)."""
        sensors = self.wrap(sensors)
        assert self.caps is not None and len(self.caps) == len(sensors), "call plan() first"
        cur = torch.cuda.current_stream(self.device)
        for st in self.streams:
            st.wait_stream(cur)
        for st in self.rstreams:
            if st is not None:
                st.wait_stream(cur)
        evs = []
        for i, s in enumerate(sensors):
            k = self.lane_of[i]
            want = times is not None or event_log is not None
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if want else None
            rs = self.rstreams[k]
            if rs is not None:   # the lane's buffers: the previous frame's render must finish first
                self.streams[k].wait_stream(rs)
            with torch.cuda.stream(self.streams[k]):
                self.lanes[k].render(s, out=outs[i], capacity=self.caps[i], events=ev,
                                     overflow=self.ovf[i:i + 1], opts=self.frame_opts[i], render_stream=rs)
            if on_frame is not None:
                fs = rs if rs is not None else self.streams[k]
                with torch.cuda.stream(fs):
                    on_frame(i, fs)
            evs.append(ev)
        if event_log is not None:
            event_log.extend(evs)
        for st in self.streams + [r for r in self.rstreams if r is not None]:
            cur.wait_stream(st)
        if times is not None:
            torch.cuda.synchronize(self.device)
            for ev in evs:
                times.project.append(ev[0].elapsed_time(ev[1]))
                times.sort.append(ev[1].elapsed_time(ev[2]))
                times.render.append(ev[2].elapsed_time(ev[3]))
        return outs

    def capture(self, sensors, outs, on_frame=None, join=()) -> "torch.cuda.CUDAGraph":
        """Capture render(sensors, outs) -- every frame's gs_project ->
        gs_bin_sort -> render launches on all lanes, with their cross-stream
        ordering -- as one CUDA graph (capacity mode has no host sync, so the
        whole batch is capturable).  Replaying it issues the batch with one
        host call instead of ~20 library calls per frame.  The lanes' buffers
        are sized by an eager render first, so nothing is allocated inside the
        capture.  Call plan() first; the graph keeps pointing at `outs` and at
        the surfel set current at capture time.  `join`: other streams
        on_frame enqueues work on (e.g. a copy stream), joined back into the
        capture at its end."""
        sensors = self.wrap(sensors)
        self.render(sensors, outs)            # eager pass: buffers at their final sizes
        torch.cuda.synchronize(self.device)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                self.render(sensors, outs, on_frame=on_frame)
                for js in join:
                    side.wait_stream(js)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        return g

    def set_surfels(self, surfels: dict):
        """Render from another device surfel set: another copy of the same set
        (a double buffer the next batch is uploaded into) keeps the planned
        capacities; a set of another size (a streamed active set) needs a new
        plan() (or render_checked)."""
        if int(surfels["means"].shape[0]) != self.n:
            self.caps = None
        for lane in self.lanes:
            lane.set_surfels(surfels)
        self.n = self.lanes[0].n

    def render_checked(self, sensors, outs, headroom: float = 1.25):
        """Render with the planned capacities, then re-render every frame
        whose pair count exceeded its capacity with a capacity grown to
        `headroom` x its exact count (one sync).  The capacity policy of a
        simulator whose poses are not known in advance: plan once, over-
        provision, and repair the rare overflow.  Returns the re-rendered
        frame indices."""
        sensors = self.wrap(sensors)
        if self.caps is None or len(self.caps) != len(sensors):
            self.plan(sensors)
        self.render(sensors, outs)
        torch.cuda.synchronize(self.device)
        bad = self.overflowed()
        lane = self.lanes[0]
        for i in bad:
            _, d_np = lane.project(sensors[i], opts=self.frame_opts[i])
            self.caps[i] = int(int(d_np.item()) * headroom) + 1
            self.ovf[i:i + 1].zero_()
            lane.render(sensors[i], out=outs[i], capacity=self.caps[i], overflow=self.ovf[i:i + 1],
                        opts=self.frame_opts[i])
        torch.cuda.synchronize(self.device)
        assert not self.overflowed()
        return bad

    def opts_of(self, i: int):
        """Options frame i of the planned batch is rendered with (None: the lane's default)."""
        return self.frame_opts[i]

    def overflowed(self):
        """Indices of frames of the last render() whose pair capacity was exceeded."""
        # one device-to-host copy; the test runs on the host (no library kernel on the GPU)
        return [i for i, v in enumerate(self.ovf.cpu().tolist()) if v]
