"""Small invocations of every libgsr.so entry point, for compute-sanitizer
(SURVEY §5).  One process, no oracle: the tools check
memory accesses, races, barrier use and initialisation, not values.

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
      python tools/sanitize_cases.py [case ...]

cases: tiny, lidar360x32, split160 (forced split lists: checkpointed merge
and re-walk), fisheye, cylindrical, decode, route, backward (default: all)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def render(s, se, **opts):
    r = Renderer(to_device(s), gsr.default_opts(**opts))
    out = r.render(se)
    torch.cuda.synchronize()
    return r, out


def main():
    cases = sys.argv[1:] or ["tiny", "lidar360x32", "split160", "fisheye", "cylindrical", "decode", "route",
                             "backward"]
    gsr.load(build_if_missing=False)
    rng = np.random.default_rng(5)
    street = sg.street(rng, 20_000, 0.0, 40.0, 3, lidar_attrs=True)
    for c in cases:
        if c == "tiny":
            t = sg.tiny()
            render(t.surfels, t.sensors[0])
        elif c == "lidar360x32":
            s = sg.street(np.random.default_rng(13), 60_000, -60.0, 60.0, 0, lidar_attrs=True, with_sh=False)
            render(s, sg.lidar64(sg.lidar_pose([0, 1.8, 0]), height=32, width=360))
        elif c == "split160":
            se = sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0))
            render(street, se, split_len=160)
            render(street, sg.lidar64(sg.lidar_pose([0, 1.8, 20.0]), height=16, width=128), split_len=160)
        elif c == "fisheye":
            k, _ = sg.draw_fisheye_k(rng, float(np.float32(np.deg2rad(95))))
            render(street, sg.fisheye(96, 80, np.deg2rad(95), k, 48.0, 40.0, sg.camera_pose([0, 1.5, 0], 0.0)))
        elif c == "cylindrical":
            render(street, sg.cylindrical(160, 64, np.deg2rad(200), np.deg2rad(60),
                                          sg.camera_pose([0, 1.5, 10.0], 0.3)))
        elif c == "decode":
            from paper_2503_11731_b200 import neural
            for modality in ("camera", "lidar"):
                a = sg.street_anchors(np.random.default_rng(3), 300, 0.0, 30.0)
                dec = sg.neural_decoder(np.random.default_rng(4), modality)
                neural.NeuralDecoder(dec, modality).decode(neural.anchors_to_device(a), [0.0, 1.5, 0.0])
            torch.cuda.synchronize()
        elif c == "route":
            from paper_2503_11731_b200 import pixdist
            se = sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0))
            pixdist.emulate(to_device(street), se, [0, 6, 12, 19], 3)
            torch.cuda.synchronize()
        elif c == "backward":
            s = sg.street(np.random.default_rng(8), 2000, 2.0, 20.0, 3, lidar_attrs=True)
            for se in (sg.pinhole(64, 48, 60.0, 32.0, 24.0, sg.camera_pose([0, 1.5, 0], 0.0)),
                       sg.lidar64(sg.lidar_pose([0, 1.8, 5.0]), height=16, width=128)):
                r, out = render(s, se, split_len=2 ** 31 - 1)
                r.backward(torch.ones_like(out))
                torch.cuda.synchronize()
        else:
            raise SystemExit(f"unknown case {c}")
        print("case", c, "ok", flush=True)


if __name__ == "__main__":
    main()
