"""Host-side cost of enqueueing frames through BatchRenderer (dev tool).
A tiny scene keeps the GPU far ahead of the host, so the enqueue time per frame
is the pure host cost (ctypes calls, launches, torch events/streams)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200.batch import BatchRenderer  # noqa: E402
from paper_2503_11731_b200.render import to_device  # noqa: E402


def main():
    surf = to_device(sg.chunked_surfels(8, 2500))   # 20k surfels
    sensors = []
    for t in range(8):
        sensors += sg.chunked_timestep_sensors(t)
    for ns in (1, 4):
        br = BatchRenderer(surf, device="cuda", n_streams=ns)
        br.plan(sensors)
        outs = br.alloc_outputs(br.wrap(sensors))
        for ev in (False, True):
            for _ in range(2):
                br.render(sensors, outs, event_log=[] if ev else None)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(5):
                br.render(sensors, outs, event_log=[] if ev else None)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            print(f"streams={ns} events={ev}: host enqueue {(t1 - t0) / (5 * len(sensors)) * 1e3:.3f} ms/frame, "
                  f"total {(t2 - t0) / (5 * len(sensors)) * 1e3:.3f} ms/frame", flush=True)


if __name__ == "__main__":
    main()
