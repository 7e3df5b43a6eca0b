"""Hottest CUDA source lines of a kernel in an ncu report (dev tool).
python tools/src_hot.py <rep> [top_n] [kernel regex]
Per line: share of executed warp instructions and of warp-stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + kf,
                     capture_output=True, text=True).stdout
rows, fname, hdr, seen_fn = [], "?", None, set()
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].rsplit("/", 1)[-1]
    elif rec[0] == "Function Name":
        if rec[1] in seen_fn and fname in [f for f, _ in seen_fn]:
            pass
    elif rec[0] == "Line No":
        hdr = rec
    elif hdr and rec[0] not in ("", "Line No"):
        try:
            smp = int(rec[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            ins = int(rec[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((fname, int(rec[0]), rec[1].strip()[:90], ins, smp))
ti = sum(r[3] for r in rows) or 1
ts = sum(r[4] for r in rows) or 1
print(f"total warp inst {ti}  stall samples {ts}")
for f, ln, src, ins, smp in sorted(rows, key=lambda r: -(r[4] / ts + r[3] / ti))[:top]:
    print(f"{f}:{ln:<5d} {ins / ti * 100:5.1f}% inst {smp / ts * 100:5.1f}% st  {src}")
