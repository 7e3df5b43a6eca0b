"""Candidates / visible surfels / pairs of Chunked frames (dev tool).
python tools/counts.py [frame indices...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def main():
    frames = [int(a) for a in sys.argv[1:]] or [224, 225, 230]
    r = Renderer(to_device(sg.chunked_surfels()))
    for fi in frames:
        se = sg.chunked_timestep_sensors(fi // 7)[fi % 7]
        r.render(se)
        torch.cuda.synchronize()
        hdr = r._last["proj"][:16].view(torch.int32).cpu().tolist()
        print({"frame": fi, "kind": int(se.kind), "n_visible": hdr[0], "n_cand": hdr[1], "pairs": r.last_pairs})


if __name__ == "__main__":
    main()
