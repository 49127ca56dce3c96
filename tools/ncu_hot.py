"""Top SASS lines by warp-stall samples from an ncu report: python tools/ncu_hot.py rep [n]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = txt.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
idx = {k: i for i, k in enumerate(h)}
k = "Warp Stall Sampling (All Samples)"
body = [x for x in rows[1:] if len(x) == len(h)]
tot = sum(float(x[idx[k]] or 0) for x in body) or 1.0
for i, x in enumerate(body):
    x.append(i)
body.sort(key=lambda x: -float(x[idx[k]] or 0))
for x in body[:n]:
    print(f"{100 * float(x[idx[k]]) / tot:5.1f}%  #{x[-1]:4d}  {x[idx['Source']].strip()[:80]}")
