"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`)
of `bench.py --steps 1 --warmup 0 --timesteps T ...`: per kernel launches,
total ms and share, over the timed step alone and over the whole command.

The timed step is located as the T*7 frames that follow the instrumented
planning pass (the last STATS compositor launch, template flag STATS = 1): each frame
starts with exactly one k_cull launch.

python tools/launch_summary.py LAUNCHES.csv TIMESTEPS [title] > summary.md
"""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    n = name.replace("void ", "").replace("gsr::", "")
    n = re.sub(r"\(.*$", "", n)
    return n


def rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    out = []
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        ns = v * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1.0)
        out.append((int(r["ID"]), short(r["Kernel Name"]), ns / 1e6))
    return out


def table(rs):
    agg = OrderedDict()
    for _, k, ms in rs:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.1f} | {100 * ms / tot:.1f}% |")
    lines.append(f"| **total (serialised, cold)** | {sum(a[0] for a in agg.values())} | {tot:.1f} | 100% |")
    return "\n".join(lines)


def main():
    path, T = sys.argv[1], int(sys.argv[2])
    title = sys.argv[3] if len(sys.argv) > 3 else path
    rs = rows(path)
    # the instrumented (STATS) compositor: k_render_pinhole<STATS, DEF>, k_render<KIND, STATS, DEF>
    stats = [i for i, (_, k, _) in enumerate(rs) if re.search(r"k_render_pinhole<1, \d>|k_render<\d, 1, \d>", k)]
    start = stats[-1] + 1 if stats else 0
    culls = [i for i in range(start, len(rs)) if rs[i][1].startswith("k_cull")]
    nfr = 7 * T
    s0 = culls[0]
    s1 = culls[nfr] if len(culls) > nfr else len(rs)
    # the last frame of the step ends before the first launch that is not part of a frame's chain
    step = rs[s0:s1]
    print(f"# {title}\n")
    print("Every kernel launch of the command, `gpu__time_duration.sum` with `--clock-control none` "
          "(ncu serialises launches and caches are cold: compare shares, not absolutes).\n")
    print(f"## The timed step alone\n\nLaunches {rs[s0][0]}..{rs[s1 - 1][0]}: the {nfr} frames of the timed step.\n")
    print(table(step))
    print("\n## The whole command\n")
    print(table(rs))


if __name__ == "__main__":
    main()
