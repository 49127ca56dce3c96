"""Timeline of sla2_attn_i8_kernel (attn_i8.cu) from the SLA2_TRACE build (analysis).

  SLA2_LIB=paper_2602_12675_b200/libsla2_i8tr.so python tools/trace_i8.py

Per CTA, lane, step g < 32 (us since lane A's first Q K^T, medians over CTAs): 0 Q K^T issued,
1 P V issued, 2 softmax has S, 10 before the absmax barrier, 9 after it, 3 P codes stored,
4 acc_PV(g - 1) visible (fold starts), 5-8 P(g) released by softmax warp 0-3."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2602_12675_b200 as sla2
    from paper_2602_12675_b200 import dist as sd
    L = sla2.lib()
    L.sla2_trace_set_buffer.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    H, N, d = 12, 32768, 128
    q, k, v, pq, pk, rho = sd.shard_inputs(0, H, 1, N, d, N // 128, torch.bfloat16, dev, 1234)
    grid = 148
    tr = torch.zeros(grid * 2 * 32 * 16, dtype=torch.int64, device=dev)
    L.sla2_trace_set_buffer(tr.data_ptr())
    for _ in range(3):
        sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True)
    torch.cuda.synchronize()
    t = tr.view(grid, 2, 32, 16).cpu().numpy().astype(np.int64)
    rel = (t - t[:, 0, 0, 0][:, None, None, None]) / 1e3
    ev = [(0, "QK iss"), (1, "PV iss"), (2, "S seen"), (10, "pre-bar"), (9, "post-bar"), (3, "codes st"),
          (4, "PV(g-1) in"), (5, "P w0"), (6, "P w1"), (7, "P w2"), (8, "P w3")]
    for x in range(2):
        print(f"lane {'AB'[x]}")
        print("  g " + "".join(f"{n:>11s}" for _, n in ev))
        for g in range(20):
            print(f" {g:2d} " + "".join(f"{np.median(rel[:, x, g, e]):11.2f}" for e, _ in ev))
    d = lambda a, b: np.median(rel[:, :, 4:20, b] - rel[:, :, 4:20, a]).round(3)
    last = rel[:, :, :, 5:9].max(axis=3)
    print("step period (last P):", np.median(np.diff(last[:, :, 4:20], axis=2)).round(3))
    print("S seen -> pre-bar:", d(2, 10), " pre -> post bar:", d(10, 9), " post-bar -> codes:", d(9, 3),
          " codes -> PV(g-1) in:", d(3, 4), " PV in -> P w0:", d(4, 5))
    print("P w0 -> PV issued:", d(5, 1), " PV issued -> next S seen:", np.median(rel[:, :, 5:21, 2] - rel[:, :, 4:20, 1]).round(3))


if __name__ == "__main__":
    main()
