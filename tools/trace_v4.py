"""Timeline of sla2_sparse_v4_kernel (sparse_v4.cu) from the SLA2_TRACE + SLA2_V4 build (analysis).

  SLA2_LIB=paper_2602_12675_b200/libsla2_v4tr.so python tools/trace_v4.py

Per CTA, query block k < 4, step j < 14 (us since block 0's PV(0), medians over CTAs): 0 PV(j)
issued, 1 softmax has S(j), 2 P(j) released, 3 QK(j+2) issued (after PV(j)). Step 14: epilogue
0 before tile_done, 1 tile_done seen, 2 lin_ready given, 3 lin_done seen, 4 O read (o_free).
Step 15: issuer 4 tile_done committed, 5 previous block's lin issued."""
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
    tr = torch.zeros(grid * 4 * 16 * 8, dtype=torch.int64, device=dev)
    L.sla2_trace_set_buffer(tr.data_ptr())
    for _ in range(3):
        sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)
    torch.cuda.synchronize()
    t = tr.view(grid, 4, 16, 8).cpu().numpy().astype(np.int64)
    rel = (t - t[:, 0, 0, 0][:, None, None, None]) / 1e3
    med = lambda a: np.median(a)
    for k in range(1, 4):
        print(f"query block {k}")
        print("   j   PV iss   S seen  P rel   QK+2")
        for j in range(15):
            print(f"  {j:2d} " + " ".join(f"{med(rel[:, k, j, e]):8.2f}" for e in range(4)))
        print("  epi: pre tile_done %.2f  tile_done %.2f  lin_ready %.2f  lin_done %.2f  o_free %.2f" %
              tuple(med(rel[:, k, 14, e]) for e in range(5)))
        print("  issuer: tile_done %.2f  prev lin issued %.2f" % (med(rel[:, k, 15, 4]), med(rel[:, k, 15, 5])))
    sp = np.diff(rel[:, 1:4, 2:14, 2], axis=2)
    print("median P spacing (steps 2-13):", med(sp).round(3), " softmax S->P:", med(rel[:, 1:4, 2:14, 2] - rel[:, 1:4, 2:14, 1]).round(3),
          " P -> PV issued:", med(rel[:, 1:4, 2:14, 0] - rel[:, 1:4, 2:14, 2]).round(3))


if __name__ == "__main__":
    main()
