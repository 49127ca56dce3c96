"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list: mean per kernel (us)."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1e-3)
            agg.setdefault(d["Kernel Name"].split("(")[0][:70], []).append(float(d["Metric Value"]) * scale)
    for n, v in agg.items():
        print(f"{n:72s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
