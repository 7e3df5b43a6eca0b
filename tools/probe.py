"""Per-stage timing and pair statistics for one frame of each config (dev tool).

python tools/probe.py [config ...]   (configs: tiny mid fisheye lidar chunked)
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


def probe(name, surfels, sensors, reps=5, opts=None, label=None):
    ct = [int(x) for x in os.environ.get("GSR_TILE", "16,8").split(",")]
    lt = [int(x) for x in os.environ.get("GSR_LTILE", "32,1").split(",")]
    r = Renderer(to_device(surfels), opts or gsr.default_opts(tile_w=ct[0], tile_h=ct[1]), lidar_tile=lt)
    res = []
    for se in sensors:
        s = gsr.Sensor(se)
        out = r.render(s)   # exact sizing, warm
        P = r.last_pairs
        stats = torch.zeros((2, se.height, se.width), dtype=torch.int32, device="cuda")
        r.render(s, capacity=P, stats=stats)
        torch.cuda.synchronize()
        st = stats.cpu().numpy().astype(np.int64)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        times = []
        for _ in range(reps):
            r.render(s, out=out, capacity=P, events=ev)
            torch.cuda.synchronize()
            times.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
        t = np.median(np.array(times), axis=0)
        nsamp = se.width * se.height
        rg = r._last["ranges"][: 2 * r._last["ntiles"]].view(-1, 2).cpu().numpy().astype(np.int64)
        ln = rg[:, 1] - rg[:, 0]
        q = np.percentile(ln, [50, 90, 99, 100]).astype(int).tolist()
        d = dict(config=label or name, kind=se.kind, W=se.width, H=se.height, n=r.n, pairs=P,
                 tiles=len(ln), list_p50_p90_p99_max=q, list_top_share=round(float(np.sort(ln)[-len(ln) // 100:].sum() / max(ln.sum(), 1)), 3),
                 ms_project=round(float(t[0]), 4), ms_sort=round(float(t[1]), 4),
                 ms_render=round(float(t[2]), 4), ms_total=round(float(t.sum()), 4),
                 msamples_per_s=round(nsamp / t.sum() / 1e3, 1),
                 contrib_per_sample=round(float(st[0].mean()), 2),
                 eval_per_sample=round(float(st[1].mean()), 2),
                 eval_max=int(st[1].max()), contrib_total=int(st[0].sum()), eval_total=int(st[1].sum()))
        print(json.dumps(d), flush=True)
        res.append(d)
    return res


def main(names):
    for name in names:
        t0 = time.time()
        if name == "chunked":
            s = sg.chunked_surfels()
            sens = sg.chunked_timestep_sensors(32)
            print(f"# chunked generated in {time.time() - t0:.1f}s", flush=True)
            probe("chunked", s, [sens[0], sens[1], sens[3], sens[6]])
        else:
            c = sg.make_config(name)
            probe(name, c.surfels, c.sensors)


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "mid", "fisheye", "lidar", "chunked"])
