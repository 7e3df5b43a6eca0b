"""Summarise an ncu report (--set full) into a per-kernel table (dev tool).

python tools/ncu_summary.py <report.ncu-rep> [out.md]

Columns: duration, DRAM bytes read+written and the achieved DRAM GB/s,
SM / issue / FMA-pipe / LSU utilisation, achieved occupancy, registers,
L1 and L2 hit rates.  Numbers come from `ncu -i ... --page raw --csv`.
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
]
SCALE = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
         "ms": 1e-3, "s": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def summarise(rep):
    h, units, data = rows(rep)
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, k in METRICS:
            if m not in h:
                continue
            i = h.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            d[k] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        if "dur" in d and "dram_rd" in d:
            d["dram_GBs"] = (d["dram_rd"] + d.get("dram_wr", 0.0)) / d["dur"] / 1e9
        res.append(d)
    return res


def to_md(res):
    cols = ["kernel", "dur_us", "dram_MB", "dram_GBs", "sm%", "issue%", "fma%", "alu%", "lsu%", "occ%", "regs",
            "l1hit%", "l2hit%"]
    lines = ["| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for d in res:
        row = [d["kernel"], f"{d.get('dur', 0) * 1e6:.1f}",
               f"{(d.get('dram_rd', 0) + d.get('dram_wr', 0)) / 1e6:.1f}", f"{d.get('dram_GBs', 0):.0f}"]
        row += [f"{d.get(k, 0):.1f}" if k != "regs" else f"{d.get(k, 0):.0f}" for k in cols[4:]]
        lines.append("| " + " | ".join(row) + " |")
    return "\n".join(lines)


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    md = to_md(res)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            f.write(md + "\n")
    print(md)
