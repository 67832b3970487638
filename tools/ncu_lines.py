"""Per-source-line and per-region breakdown of an ncu --import-source capture.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [top_n]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
hdr = None
lines = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or not r[0].isdigit():
        continue
    try:
        s, i = int(r[4]), int(r[7])
    except ValueError:
        continue
    lines.append((s, i, cur, int(r[0]), r[1].strip()[:80]))
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"samples {ts}  warp-instructions {ti:,}")
for s, i, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{s / ts * 100:5.1f}%s {i / ti * 100:5.1f}%i  {f}:{ln}  {src}")
