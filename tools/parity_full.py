"""Full-frame parity statistics, GPU vs oracle, on the GPU box (BASELINE.md §3,
VERDICT r1 item 2): every pixel of the Tiny, Mid, Fisheye and LiDAR frames and
4096 random rays of each of the 14 frames of Chunked timesteps 0 and 32,
rendered exactly as bench.py renders them, under the strict two-sided gate of
tests/parity.py.  Writes per frame: rays, flagged / ambiguous / bad counts,
per-channel max / p99.99 / mean |delta| on unflagged rays, oracle seconds and
threads.

python tools/parity_full.py OUT.json [tiny mid fisheye lidar chunked]
(test infrastructure: runs the oracle; never part of the product path)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import scenegen as sg  # noqa: E402
from paper_2503_11731_b200.batch import BatchRenderer  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402
from tests import parity  # noqa: E402


def check(surfels, se, img, rays, label):
    cores = len(os.sched_getaffinity(0))
    t = time.time()
    ref, fl, _ = oracle.render(surfels, se, rays, nthreads=cores)
    t_or = time.time() - t
    st = parity.compare(img, ref, fl, rays, se, surfels)
    st["oracle_s"] = round(t_or, 1)
    st["oracle_threads"] = cores
    st["ambiguous_cap"] = max(2, parity.MAX_AMBIGUOUS_FRAC * len(rays))
    st["flag_bits"] = {str(b): int(((fl & b) != 0).sum()) for b in (1, 2, 4, 8, 16, 32, 64)}
    print(label, {k: v for k, v in st.items() if k != "per_channel_unflagged"}, flush=True)
    return st


def main():
    out = sys.argv[1]
    which = sys.argv[2:] or ["tiny", "mid", "lidar", "fisheye", "chunked"]
    res = json.load(open(out)) if os.path.exists(out) else {}
    res["_about"] = ("tools/parity_full.py: GPU (libgsr.so) vs the fp64 oracle, strict gate of tests/parity.py; "
                     "full frames for tiny/mid/lidar/fisheye, 4096 random rays x 14 frames for chunked")
    for name in which:
        if name == "chunked":
            s = sg.chunked_surfels()
            dev = to_device(s)
            for t in (0, 32):
                sensors = sg.chunked_timestep_sensors(t)
                br = BatchRenderer(dev, n_streams=4)   # the bench's renderer: capacity mode, per-frame tiles
                br.plan(sensors)
                outs = br.alloc_outputs(br.wrap(sensors))
                br.render(sensors, outs)
                torch.cuda.synchronize()
                assert br.overflowed() == []
                for i, se in enumerate(sensors):
                    rng = np.random.default_rng(1000 * t + i)
                    rays = np.sort(rng.choice(se.width * se.height, 4096, replace=False)).astype(np.int64)
                    key = f"chunked_t{t}_s{i}"
                    res[key] = check(s, se, outs[i].cpu().numpy(), rays, key)
                    json.dump(res, open(out, "w"), indent=1)
            del dev
        else:
            c = sg.make_config(name)
            se = c.sensors[0]
            img = Renderer(to_device(c.surfels)).render(se).cpu().numpy()
            rays = np.arange(se.width * se.height, dtype=np.int64)
            res[name] = check(c.surfels, se, img, rays, name)
            json.dump(res, open(out, "w"), indent=1)
        torch.cuda.empty_cache()
    tot = {k: sum(v[k] for n, v in res.items() if not n.startswith("_")) for k in
           ("n", "flagged", "ambiguous", "bad", "bad_flagged", "unresolved")}
    tot["ok_all"] = all(v["ok"] for n, v in res.items() if not n.startswith("_"))
    res["_total"] = tot
    json.dump(res, open(out, "w"), indent=1)
    print("total", tot)


if __name__ == "__main__":
    main()
