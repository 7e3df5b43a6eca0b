"""Render one frame of a config a few times (for ncu captures).

python tools/one_frame.py <config> [frame_index] [reps]
config: tiny mid fisheye lidar chunked (chunked frame index 0..447)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "mid"
    fi = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    if name == "chunked":
        s = sg.chunked_surfels()
        sensor = sg.chunked_timestep_sensors(fi // 7)[fi % 7]
    else:
        c = sg.make_config(name)
        s, sensor = c.surfels, c.sensors[fi]
    r = Renderer(to_device(s))
    gs = gsr.Sensor(sensor)
    out = r.render(gs)
    P = r.last_pairs
    for _ in range(reps):
        r.render(gs, out=out, capacity=P)
    torch.cuda.synchronize()
    print(name, fi, "pairs", P, "alpha_mean", float(out[-1].mean()))


if __name__ == "__main__":
    main()
