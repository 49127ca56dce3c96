"""Pipeline timeline of the sparse kernel from the SLA2_TRACE build (analysis only).

  SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so python tools/trace_sparse.py

Prints, over all CTAs of one cfg2 forward, the median per-CTA durations of the phases:
prologue (start -> Q ready), each key block's S-ready / P-ready times, the loop, and the
epilogue steps, plus how CTAs of consecutive waves overlap on the device clock."""
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
    L.sla2_trace_set_buffer.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    B, H, N, d = 1, int(os.environ.get("H", "12")), 32768, 128
    tm = N // 128
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((B, H, N, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    eye = torch.eye(d, device=dev)[None]
    pq = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    pk = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    rho = torch.zeros((H, tm), device=dev)
    tr = torch.zeros(B * H * tm * 128, dtype=torch.int64, device=dev)
    L.sla2_trace_set_buffer(tr.data_ptr())
    for _ in range(3):
        sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)
    torch.cuda.synchronize()
    t = tr.view(B * H * tm, 128).cpu().numpy().astype(np.int64)
    t0 = t[:, 0]
    rel = (t - t0[:, None]) / 1000.0  # us since CTA start
    kappa = 15

    def med(x):
        return float(np.median(x))
    print(f"CTAs {len(t)}  kernel span {(t[:, 53].max() - t0.min()) / 1e3:.1f} us")
    print(f"per-CTA total (start -> output done): median {med(rel[:, 53]):.2f} us")
    print(f"  Q ready at MMA         {med(rel[:, 1]):7.2f}")
    print(f"  producer first/last kv {med(rel[:, 54]):7.2f} / {med(rel[:, 55]):7.2f}")
    for j in range((kappa + 1) // 2):  # key-block pairs
        print(f"  pair {j:2d}: K ready {med(rel[:, 56 + j]):7.2f}  S ready {med(rel[:, 2 + j]):7.2f}"
              f"  P ready {med(rel[:, 18 + j]):7.2f}  PV issued {med(rel[:, 34 + j]):7.2f}")
    for j in range(kappa):
        print(f"  V {j:2d}: load issued {med(rel[:, 64 + j]):7.2f}  ready at MMA {med(rel[:, 80 + j]):7.2f}"
              f"  (latency {med(rel[:, 80 + j] - rel[:, 64 + j]):5.2f})  arrived {med(rel[:, 96 + j]):7.2f}")
    for n in range((kappa + 1) // 2):
        print(f"  pair {n}: HS issued {med(rel[:, 112 + n]):7.2f}")
    print(f"  loop done (pv_done)    {med(rel[:, 50]):7.2f}")
    print(f"  lin_ready              {med(rel[:, 51]):7.2f}")
    print(f"  lin_done               {med(rel[:, 52]):7.2f}")
    print(f"  output done            {med(rel[:, 53]):7.2f}")
    starts = np.sort(t0)
    print(f"start spread: first {0:.1f}, 148th {(starts[147] - starts[0]) / 1e3:.1f} us, "
          f"296th {(starts[295] - starts[0]) / 1e3:.1f} us, last {(starts[-1] - starts[0]) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
