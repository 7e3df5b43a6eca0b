"""Render the BASELINE configs on the GPU and save sampled GPU outputs
(ray indices + values) to an .npz per frame, for offline parity analysis
against the oracle on the dev box (the oracle is not run here).

python tools/dump_gpu.py OUTDIR [which ...]
which: mid fisheye lidar chunked   (default: all)
python tools/dump_gpu.py OUTDIR full CONFIG ROW0 ROW1
    all pixels of rows [ROW0, ROW1) of the config's frame (full-frame parity
    in slabs small enough for gpurun_out)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200.batch import BatchRenderer  # noqa: E402
from paper_2503_11731_b200.render import Renderer, to_device  # noqa: E402


def sample(se, n, seed):
    rng = np.random.default_rng(seed)
    tot = se.width * se.height
    return np.sort(rng.choice(tot, min(n, tot), replace=False)).astype(np.int64)


def save(outdir, name, img, rays):
    C = img.shape[0]
    vals = img.reshape(C, -1)[:, rays].T.copy()
    np.savez(os.path.join(outdir, name + ".npz"), rays=rays, gpu=vals)
    print(name, img.shape, len(rays), flush=True)


def main():
    outdir = sys.argv[1]
    os.makedirs(outdir, exist_ok=True)
    if len(sys.argv) > 2 and sys.argv[2] == "full":
        name, r0, r1 = sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
        c = sg.make_config(name)
        se = c.sensors[0]
        img = Renderer(to_device(c.surfels)).render(se).cpu().numpy()
        r1 = min(r1, se.height)
        rays = np.arange(r0 * se.width, r1 * se.width, dtype=np.int64)
        save(outdir, f"{name}_full_{r0}_{r1}", img, rays)
        return
    which = sys.argv[2:] or ["mid", "fisheye", "lidar", "chunked"]
    for name in which:
        if name == "chunked":
            s = sg.chunked_surfels()
            dev = to_device(s)
            for t in (0, 32, 63):
                sensors = sg.chunked_timestep_sensors(t)
                br = BatchRenderer(dev, n_streams=2)
                br.plan(sensors)
                outs = br.alloc_outputs(br.wrap(sensors))
                br.render(sensors, outs)
                torch.cuda.synchronize()
                assert br.overflowed() == []
                for i, se in enumerate(sensors):
                    save(outdir, f"chunked_t{t}_s{i}", outs[i].cpu().numpy(), sample(se, 20000, 1000 * t + i))
            del dev
        else:
            c = sg.make_config(name)
            se = c.sensors[0]
            img = Renderer(to_device(c.surfels)).render(se).cpu().numpy()
            n = se.width * se.height if name == "lidar" else 300_000
            save(outdir, name, img, sample(se, n, 7))
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
