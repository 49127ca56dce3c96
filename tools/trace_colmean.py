"""Per-chunk timeline of the exact column-mean kernel (trace build, analysis only).

  SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so python tools/trace_colmean.py"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2602_12675_b200 as sla2
    L = sla2.lib()
    L.sla2_cm_trace_set.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    B, H, N, d = 1, 12, 32768, 128
    k = torch.randn((B, H, N, d), device=dev).to(torch.bfloat16)
    mu = torch.empty((B * H, d), device=dev)
    tr = torch.zeros(1024, dtype=torch.int64, device=dev)
    L.sla2_cm_trace_set(tr.data_ptr())
    for _ in range(3):
        sla2.smooth_k(k)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    n = N // 128
    dt = np.diff(t[: n - 1]) / 1000.0
    print(f"chunks {n - 1}: span {(t[n - 2] - t[0]) / 1e3:.1f} us, per chunk median {np.median(dt):.3f} us, "
          f"p90 {np.percentile(dt, 90):.3f}, max {dt.max():.3f}; ideal 128 rows x 4 cycles = "
          f"{128 * 4 / 1.965e3:.3f} us")
    print("first 24 chunk gaps:", " ".join(f"{x:.2f}" for x in dt[:24]))
    print("slowest 10 at:", np.argsort(dt)[-10:])


if __name__ == "__main__":
    main()
