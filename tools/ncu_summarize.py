"""Summarise ncu captures into profiles/ (analysis only).

  python tools/ncu_summarize.py full <report.ncu-rep> <out.txt> [--config cfg2 --summary profiles/ncu_summary.json]
  python tools/ncu_summarize.py launches <launches.csv> <out.txt>

`full`: per-kernel duration, DRAM bytes (read + write, the bench line's roofline.traffic),
L2 bytes, tensor-pipe activity, SM throughput and issue activity from a `--set full` report;
with --summary it also records the sparse kernel's DRAM bytes per launch for bench.py.
`launches`: per-kernel launch counts and mean durations from a `--metrics
gpu__time_duration.sum` CSV, with each kernel's share of the listed time."""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("gpc__cycles_elapsed.max", "cycles"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def full(rep, out, config=None, summary=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    lines = [f"ncu --set full summary of {rep}", ""]
    sparse_bytes = None
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        name = d.get("Kernel Name", "?")
        lines.append(f"== {name[:110]}")
        vals = {}
        for k, label in KEYS:
            if k not in d:
                continue
            v = d[k].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                lines.append(f"   {label:24s} {v} {u.get(k, '')}")
                continue
            vals[k] = x * SCALE.get(u.get(k, ""), 1)
            lines.append(f"   {label:24s} {x:,.3f} {u.get(k, '')}")
        if "dram__bytes_read.sum" in vals and "dram__bytes_write.sum" in vals:
            tot = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
            lines.append(f"   {'dram read+write':24s} {tot / 1e6:,.1f} MB")
            if "sla2_sparse_bf16" in name:
                sparse_bytes = tot
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("\n".join(lines))
    if summary and config and sparse_bytes is not None:
        try:
            s = json.load(open(summary))
        except (OSError, ValueError):
            s = {}
        s.setdefault(config, {})["sparse_kernel_dram_bytes_per_launch"] = int(sparse_bytes)
        s[config]["source"] = rep.split("/")[-1] + " (ncu --set full, one launch)"
        json.dump(s, open(summary, "w"), indent=1)


def launches(csvf, out):
    rows = list(csv.reader(open(csvf)))
    i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    head = rows[i]
    agg = OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(head, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:90]
        ns = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Unit") == "usecond":
            ns *= 1e3
        agg.setdefault(name, []).append(ns)
    total = sum(sum(v) for v in agg.values())
    lines = [f"kernel launch list of {csvf} (ncu --metrics gpu__time_duration.sum --clock-control none;",
             "cold-cache, serialised: compare shares, not absolutes)", "",
             f"{'kernel':90s} {'n':>4s} {'mean us':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
        lines.append(f"{k:90s} {len(v):4d} {sum(v) / len(v) / 1e3:9.1f} {sum(v) / total:6.1%}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        a = sys.argv[2:]
        cfg = a[a.index("--config") + 1] if "--config" in a else None
        sm = a[a.index("--summary") + 1] if "--summary" in a else None
        full(a[0], a[1], cfg, sm)
    else:
        launches(sys.argv[2], sys.argv[3])
