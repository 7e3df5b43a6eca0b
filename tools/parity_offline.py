"""Parity statistics from GPU dumps (tools/dump_gpu.py) against the oracle,
computed on the dev box: per frame the strict two-sided gate of
tests/parity.py, with per-channel max / p99.99 / mean and flagged counts.

python tools/parity_offline.py DUMPDIR OUT.json [which ...] [--chunked-rays N]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import scenegen as sg  # noqa: E402
from tests import parity  # noqa: E402


def frame(surfels, se, dump, nmax, label):
    d = np.load(dump)
    rays, gpu = d["rays"], d["gpu"]
    if nmax and len(rays) > nmax:
        keep = np.sort(np.random.default_rng(0).choice(len(rays), nmax, replace=False))
        rays, gpu = rays[keep], gpu[keep]
    C = gpu.shape[1]
    img = np.zeros((C, se.width * se.height), np.float32)
    img[:, rays] = gpu.T
    t = time.time()
    ref, fl, _ = oracle.render(surfels, se, rays)
    st = parity.compare(img.reshape(C, se.height, se.width), ref, fl, rays, se, surfels)
    st["oracle_s"] = round(time.time() - t, 1)
    st["flag_bits"] = {str(b): int(((fl & b) != 0).sum()) for b in (1, 2, 4, 8, 16, 32, 64)}
    print(label, {k: v for k, v in st.items() if k not in ("per_channel_unflagged",)}, flush=True)
    return st


def main():
    dump, out = sys.argv[1], sys.argv[2]
    args = [a for a in sys.argv[3:] if not a.startswith("--")]
    nchunk = 2000
    for a in sys.argv[3:]:
        if a.startswith("--chunked-rays="):
            nchunk = int(a.split("=")[1])
    which = args or ["mid", "fisheye", "lidar", "chunked"]
    res = json.load(open(out)) if os.path.exists(out) else {}
    for name in which:
        if name == "chunked":
            s = sg.chunked_surfels()
            for t in (0, 32, 63):
                sensors = sg.chunked_timestep_sensors(t)
                for i, se in enumerate(sensors):
                    key = f"chunked_t{t}_s{i}"
                    p = os.path.join(dump, key + ".npz")
                    if os.path.exists(p):
                        res[key] = frame(s, se, p, nchunk, key)
                        json.dump(res, open(out, "w"), indent=1)
        else:
            c = sg.make_config(name)
            res[name] = frame(c.surfels, c.sensors[0], os.path.join(dump, name + ".npz"), 0, name)
            json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
