"""Timeline of sla2_attn_kernel (sparse_fa.cu) from the SLA2_TRACE build (analysis).

  SLA2_LIB=paper_2602_12675_b200/libsla2_fatr.so python tools/trace_fa.py [dense]

Per CTA, lane and step g < 32: 0 Q K^T(g) issued, 1 P V(g) issued, 2 softmax has S(g), 3 P(g)
arrived, 4 K(g) load issued, 5 V(g) load issued. Prints medians over CTAs (us, relative to lane
A's first Q K^T) and per-step gaps."""
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
    dense = len(sys.argv) > 1 and sys.argv[1] == "dense"
    L = sla2.lib()
    L.sla2_trace_set_buffer.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    H, N, d = 12, 32768, 128
    tm = N // 128
    q, k, v, pq, pk, rho = sd.shard_inputs(0, H, 1, N, d, tm, torch.bfloat16, dev, 1234)
    grid = 148
    tr = torch.zeros(grid * 2 * 32 * 16, dtype=torch.int64, device=dev)
    L.sla2_trace_set_buffer(tr.data_ptr())
    for _ in range(3):
        if dense:
            sla2.full_attention(q[:, :2], k[:, :2], v[:, :2])
        else:
            sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)
    torch.cuda.synchronize()
    t = tr.view(grid, 2, 32, 16).cpu().numpy().astype(np.int64)
    base = t[:, 0, 0, 0][:, None, None]
    rel = (t - base[..., None]) / 1e3
    names = ["QK issued", "PV issued", "S seen", "P w0", "P w1", "P w2", "P w3", "P seen"]
    for x in range(2):
        print(f"lane {'AB'[x]}: median us since lane A QK(0)")
        print("  g  " + "".join(f"{n:>11s}" for n in names))
        for g in range(32):
            row = [np.median(rel[:, x, g, e]) for e in range(8)]
            print(f"  {g:2d} " + "".join(f"{v:11.2f}" for v in row))
    last = rel[:, :, :, 3:7].max(axis=3)
    print("median P (last warp) spacing per lane step:", np.median(np.diff(last, axis=2)[:, :, 4:]).round(3))
    print("median softmax warp spread (last - first P arrival):", np.median(last[:, :, 4:] - rel[:, :, 4:, 3:7].min(axis=3)).round(3))
    print("median last P arrival -> issuer saw P:", np.median(rel[:, :, 4:, 7] - last[:, :, 4:]).round(3))
    for e, nm in ((8, "LDTM done"), (9, "max done"), (10, "exp done"), (11, "STTM done"), (3, "P arrived")):
        print(f"median S seen -> {nm}:", np.median(rel[:, :, 4:, e] - rel[:, :, 4:, 2]).round(3))
    print("median S seen -> P w0:", np.median(rel[:, :, 4:, 3] - rel[:, :, 4:, 2]).round(3))


if __name__ == "__main__":
    main()
