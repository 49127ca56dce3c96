"""Warp-stall samples per CUDA source line (analysis): ncu SASS page x nvdisasm -g line table.
  python tools/ncu_lines.py report.ncu-rep build/obj.o kernel_substring [n]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
# one block per profiled launch ("Kernel Name" line, header, rows): INST picks the launch
starts = [k for k, ln in enumerate(lines) if ln.startswith('"Kernel Name"')] or [0]
inst = int(os.environ.get("INST", "0"))
lo = starts[inst]
hi = starts[inst + 1] if inst + 1 < len(starts) else len(lines)
rows = list(csv.reader(io.StringIO("\n".join(lines[lo + 1:hi]))))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
body = [r for r in rows[1:] if len(r) == len(h)]
samples = [(r[ix["Source"]].strip(), float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)) for r in body]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    g = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
# the kernel's instructions in order with their source line
insts = []
cur = None
infun = False
for line in g.splitlines():
    if re.match(r"\s*\.text\.", line) or line.startswith(".text"):
        infun = os.environ.get("KDIS", kern) in line
    ms = re.findall(r"(\w+\.cuh?)\", line (\d+)", line)
    if ms and "//##" in line:  # outermost caller of inlined code
        cur = ms[-1][0] + ":" + ms[-1][1]
    if infun and re.search(r"/\*[0-9a-f]{4,}\*/", line):
        insts.append(cur)
tot = sum(s for _, s in samples) or 1
if len(insts) != len(samples):
    print(f"warning: {len(insts)} disassembled vs {len(samples)} profiled instructions")
c = collections.Counter()
for (src, s), ln in zip(samples, insts):
    c[ln] += s
for ln, s in c.most_common(n):
    print(f"{100 * s / tot:5.1f}%  {ln}")
# stall reasons over source-line ranges: RANGES="softmax=sparse_v3.cu:460-545,epi=..."
for spec in filter(None, os.environ.get("RANGES", "").split(",")):
    name, rng = spec.split("=")
    f, lr = rng.split(":")
    lo, hi = (int(x) for x in lr.split("-"))
    agg = collections.Counter()
    for r, ln in zip(body, insts):
        if ln and ln.startswith(f + ":") and lo <= int(ln.split(":")[1]) <= hi:
            for k in reasons:
                agg[k] += float(r[ix[k]] or 0)
    t = sum(agg.values()) or 1
    print(name, f"{100 * t / tot:.1f}% of samples:", ", ".join(f"{k[6:]} {100 * v / t:.0f}%" for k, v in agg.most_common(8)))
