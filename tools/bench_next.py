"""Throughput of the SURVEY §8(f) NEXT components on one B200 (dev tool;
its JSON lines are summarised in profiles/ and DESIGN.md §12-§15).

  backward   gs_render_backward on the Mid frame (200 K surfels, 1920x1080,
             pinhole) and the LiDAR config sweep (2 M surfels, 64x2048):
             forward and backward ms (CUDA events, median of 5).
  stream     the Chunked trajectory (64 timesteps x 7 frames) rendered from
             per-pose active sets (zones with 25 % padding,
             double-buffered uploads on a copy stream, swap when complete)
             instead of the whole 12 M-surfel replica: Msamples/s, upload
             bytes, swaps, time the host waited for an upload.

python tools/bench_next.py [backward] [stream]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def med_ms(fn, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def backward():
    for name in ("mid", "lidar"):
        c = sg.make_config(name)
        se = c.sensors[0]
        r = Renderer(to_device(c.surfels), gsr.default_opts(split_len=2 ** 31 - 1))
        out = r.render(se)
        torch.cuda.synchronize()
        P = r.last_pairs
        g = torch.from_numpy(np.random.default_rng(0).normal(size=tuple(out.shape)).astype(np.float32)).cuda()
        r.backward(g)
        torch.cuda.synchronize()
        fwd = med_ms(lambda: r.render(se, out=out, capacity=P))
        bwd = med_ms(lambda: r.backward(g))
        npx = se.width * se.height
        print(json.dumps({"what": "backward", "config": name, "surfels": c.surfels.n, "frame": f"{se.width}x{se.height}",
                          "pairs": P, "ms_forward_unsplit": round(fwd, 3), "ms_backward": round(bwd, 3),
                          "backward_Msamples_s": round(npx / (bwd * 1e-3) / 1e6, 1)}), flush=True)


def stream():
    from paper_2503_11731_b200.batch import BatchRenderer
    from paper_2503_11731_b200.stream import ChunkStreamer, chunked_zones
    chunks = [sg.street(np.random.default_rng(100 + c), 1_500_000, 50.0 * c, 50.0 * c + 50.0, 3, lidar_attrs=True)
              for c in range(8)]
    st = ChunkStreamer(chunks, chunked_zones())
    T = 64
    poses = [sg.chunked_timestep_sensors(t) for t in range(T)]
    z = lambda t: 168.0 + t
    st.load((0.0, 1.5, z(0)))
    br = BatchRenderer(st.front(), n_streams=10, grid_share=0.2)
    outs = br.alloc_outputs(br.wrap(poses[0]))
    # warm-up: one pass over a few timesteps
    for t in range(3):
        br.set_surfels(st.front())
        br.render_checked(poses[t], outs)
    torch.cuda.synchronize()
    st.poll(wait=True)
    st2 = st
    st2.load((0.0, 1.5, z(0)))
    st2.bytes_uploaded, st2.swaps = 0, 0
    br.set_surfels(st2.front())
    wait_s = 0.0
    sets = []
    rerenders = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    for t in range(T):
        st2.update((0.0, 1.5, z(t)))
        tw = time.perf_counter()
        st2.poll()             # swap if the back buffer is complete (no wait)
        wait_s += time.perf_counter() - tw
        br.set_surfels(st2.front())
        sets.append(st2.front_set())
        rerenders += len(br.render_checked(poses[t], outs))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    samples = sum(s.width * s.height for p in poses for s in p)
    print(json.dumps({"what": "stream", "timesteps": T, "frames": 7 * T, "ms_total": round(ms, 1),
                      "Msamples_s": round(samples / (ms * 1e-3) / 1e6, 1),
                      "wall_s": round(time.perf_counter() - t0, 2),
                      "bytes_uploaded": st2.bytes_uploaded, "swaps": st2.swaps,
                      "active_sets": sorted({str(s) for s in sets}),
                      "buffer_capacity_surfels": st2.capacity, "capacity_rerenders": rerenders,
                      "host_poll_s": round(wait_s, 4),
                      "note": "render_checked syncs once per timestep (capacity repair); sets change size"}),
          flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["backward", "stream"]
    gsr.load()
    for w in which:
        globals()[w]()
