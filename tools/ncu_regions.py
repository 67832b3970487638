"""Aggregate an ncu --import-source capture by line ranges: ncu_regions.py rep file:lo-hi=name ..."""
import csv
import subprocess
import sys

rep = sys.argv[1]
regions = []
for spec in sys.argv[2:]:
    loc, name = spec.split("=")
    f, rng = loc.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    regions.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
agg = {}
ts = ti = 0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r[0].isdigit():
        continue
    try:
        s, i = int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    ln = int(r[0])
    name = "other:" + cur
    for f, lo, hi, nm in regions:
        if f == cur and lo <= ln <= hi:
            name = nm
            break
    a = agg.setdefault(name, [0, 0])
    a[0] += s
    a[1] += i
    ts += s
    ti += i
for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} samples {s / ts * 100:5.1f}%  instr {i / ti * 100:5.1f}%  ({i:,})")
