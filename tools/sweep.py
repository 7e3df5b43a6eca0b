"""Sweep render settings (tile shape, warp layout, split length) per frame (dev tool).

python tools/sweep.py <config> [cam_tiles] [lidar_tiles] [unused] [split_lens]
  config: mid fisheye lidar tiny chunked (chunked: t=32 forward, side, LiDAR)
  cam_tiles / lidar_tiles: e.g. 16x16,32x16 ; split_lens: 0,4096 (0 = adaptive)
  (the fourth argument once selected an experimental warp layout; it is ignored)
Prints one JSON line per (frame, setting): ms per stage (median of 5).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def parse_tiles(s):
    return [tuple(int(v) for v in t.split("x")) for t in s.split(",")]


def main():
    name = sys.argv[1]
    cam_tiles = parse_tiles(sys.argv[2]) if len(sys.argv) > 2 else [(16, 16)]
    lid_tiles = parse_tiles(sys.argv[3]) if len(sys.argv) > 3 else [(64, 4)]
    layouts = [int(v) for v in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0]
    splits = [int(v) for v in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0]
    if name == "chunked":
        s = sg.chunked_surfels()
        se = sg.chunked_timestep_sensors(32)
        frames = [("fwd", se[0]), ("side", se[1]), ("lidar", se[6])]
    else:
        c = sg.make_config(name)
        s = c.surfels
        frames = [(name, c.sensors[0])]
    dev = to_device(s)
    for label, sensor in frames:
        gs = gsr.Sensor(sensor)
        tiles = lid_tiles if sensor.kind == gsr.GS_LIDAR_SPINNING else cam_tiles
        for (tw, th) in tiles:
            for lay in layouts:
                for L in splits:
                    opts = gsr.default_opts(tile_w=tw, tile_h=th, split_len=L)
                    r = Renderer(dev, opts, lidar_tile=(tw, th))
                    out = r.render(gs)
                    P = r.last_pairs
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    ts = []
                    for _ in range(5):
                        r.render(gs, out=out, capacity=P, events=ev)
                        torch.cuda.synchronize()
                        ts.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
                    t = np.median(np.array(ts), axis=0)
                    print(json.dumps(dict(frame=label, tile=f"{tw}x{th}", layout=lay, split=L, pairs=P,
                                          ms_project=round(float(t[0]), 3), ms_sort=round(float(t[1]), 3),
                                          ms_render=round(float(t[2]), 3), ms_total=round(float(t.sum()), 3),
                                          alpha_mean=round(float(out[-1].mean()), 5))), flush=True)
                    del r


if __name__ == "__main__":
    main()
