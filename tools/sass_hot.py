"""Hottest SASS instructions of a kernel in an ncu report (dev tool).
python tools/sass_hot.py <rep> [min_frac] [kernel regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf,
                     capture_output=True, text=True).stdout
lines = out.splitlines()
ends = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
lines = lines[1:ends[1]] if len(ends) > 1 else lines[1:]   # first captured launch only
r = list(csv.reader(io.StringIO("\n".join(lines))))
h = r[0]
ie = h.index("Instructions Executed"); src = h.index("Source"); st = h.index("Warp Stall Sampling (All Samples)")
rows = [(x[0], x[src], int(x[ie] or 0), int(x[st] or 0)) for x in r[1:] if len(x) > ie]
tot = sum(x[2] for x in rows); tst = sum(x[3] for x in rows)
print("total inst", tot, "samples", tst)
for a, s, n, smp in rows:
    if n >= mn * tot or smp >= 0.01 * tst:
        print(f"{a[-5:]} {n / tot * 100:5.1f}% {smp / max(tst,1) * 100:5.1f}%st {s.strip()}")
