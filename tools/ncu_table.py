"""Per-kernel table of several ncu raw exports (dev tool): duration, DRAM bytes,
achieved DRAM GB/s and its fraction of the measured HBM peak
(MEASURED_PEAKS.json hbm_gbs), issue / FMA-pipe utilisation, occupancy.

python tools/ncu_table.py TITLE RAW.csv[:label] ... > table.md
(RAW.csv = `ncu -i rep --page raw --csv`; the first frame's launches, in order.)
"""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
M = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
     "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "fma": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "occ": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread"}


def load(path):
    """Launches of the first frame in the export (up to the second k_cull), in order."""
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    out = OrderedDict()
    seen_cull = False
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("gsr::", "").strip()
        if name.startswith("k_cull"):
            if seen_cull:
                break
            seen_cull = True
        if name in out or any(k.startswith(name + " #") for k in out):
            k = 2
            while f"{name} #{k}" in out:
                k += 1
            if name in out:
                out[name + " #1"] = out.pop(name)
            name = f"{name} #{k}"
        d = {}
        for k, m in M.items():
            if m in h:
                i = h.index(m)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(u[i], 1.0)
                except ValueError:
                    pass
        out.setdefault(name, []).append(d)
    return out


def main():
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(f"# {sys.argv[1]}\n")
    print(f"HBM peak {peak:.0f} GB/s (MEASURED_PEAKS.json).  ncu `--set full --clock-control none`: cold caches, "
          "serialised launches; one frame's launches in order (#k: the k-th launch of a kernel).\n")
    for arg in sys.argv[2:]:
        path, _, label = arg.partition(":")
        print(f"## {label or os.path.basename(path)}\n")
        print("| kernel | launches | us / launch | DRAM MB / launch | GB/s | % of HBM peak | issue % | FMA pipe % | occupancy % | regs |")
        print("|---|---|---|---|---|---|---|---|---|---|")
        tot = 0.0
        for name, ds in load(path).items():
            n = len(ds)
            avg = lambda k: sum(d.get(k, 0.0) for d in ds) / n
            dur, byt = avg("dur"), avg("rd") + avg("wr")
            gbs = byt / dur / 1e9 if dur > 0 else 0.0
            tot += dur * n
            print(f"| `{name}` | {n} | {dur * 1e6:.1f} | {byt / 1e6:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f} | "
                  f"{avg('issue'):.1f} | {avg('fma'):.1f} | {avg('occ'):.1f} | {avg('regs'):.0f} |")
        print(f"\ntotal {tot * 1e3:.3f} ms\n")


if __name__ == "__main__":
    main()
