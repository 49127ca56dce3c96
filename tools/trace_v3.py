"""Timeline of the persistent sparse kernel (sparse_v3.cu) from the SLA2_TRACE build (analysis).

  SLA2_LIB=paper_2602_12675_b200/libsla2_b200_trace.so python tools/trace_v3.py

Per CTA and tile k (k < 8) the kernel stamps %globaltimer at: 0 MMA has the tile's Q; 1-8 S of
pair n ready (softmax half 0); 9-16 P of pair n written (half 0); 28 S pair 0 ready (half 1);
31 softmax tile end; 17 epilogue sees the tile's last MMA; 18 O stashed (o_free); 19 lin_ready;
20 lin_done seen; 21 output stored (hl_free); 22 issuer: lin MMA issued; 23 issuer: hl_free seen;
24 issuer: tile done; 25/26/27 PV of pair 0/1/last issued; 29 epilogue: zc seen; 30 sm_done seen.
Prints medians (us) relative to the tile's stamp 0 for tiles 1..6 (steady state)."""
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
    B, H, N, d = 1, int(os.environ.get("H", "12")), int(os.environ.get("N", "32768")), 128
    kp = float(os.environ.get("KP", "3.0"))
    tm = -(-N // 128)
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((B, H, N, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    eye = torch.eye(d, device=dev)[None]
    pq = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    pk = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    rho = torch.zeros((H, tm), device=dev)
    grid = 148
    tr = torch.zeros(grid * 8 * 96, dtype=torch.int64, device=dev)
    L.sla2_trace_set_buffer(tr.data_ptr())
    for _ in range(3):
        sla2.forward(q, k, v, pq, pk, rho, k_percent=kp)
    torch.cuda.synchronize()
    t = tr.view(grid, 8, 96).cpu().numpy().astype(np.int64)
    names = {0: "Q ready (MMA)", 17: "epi: tile MMAs done", 18: "epi: O stashed", 19: "epi: lin_ready",
             20: "epi: lin_done", 21: "epi: stored", 22: "MMA: lin issued", 23: "MMA: hl_free seen",
             24: "MMA: tile done", 25: "MMA: PV pair 0", 26: "MMA: PV pair 1", 27: "MMA: PV last pair",
             28: "S ready pair 0 (h1)", 29: "epi: zc seen", 30: "epi: sm_done seen", 31: "softmax tile end"}
    for n in range(8):
        names[1 + n] = f"S ready pair {n}"
        names[9 + n] = f"P ready pair {n}"
        names[32 + n] = f"MMA: p_full {n} seen"
        names[40 + n] = f"MMA: PV {n} issued"
        names[48 + n] = f"MMA: QK {n + 2} issued"
        names[56 + n] = f"MMA: Hsel {n} issued"
        names[64 + n] = f"TMA: K pair {n} issued"
        names[72 + n] = f"TMA: V block {2 * n + 1} issued"
        names[80 + n] = f"MMA: PV {n} start (before V wait)"
        names[88 + n] = f"MMA: QK {n + 2} start (before K wait)"
    ks = range(1, 7)
    base = t[:, ks, 0]
    print(f"median per-tile (us since the tile's Q ready), tiles {list(ks)}, {grid} CTAs")
    for e in sorted(names):
        x = t[:, ks, e]
        ok = x > 0
        if ok.sum() == 0:
            continue
        rel = (x - base)[ok] / 1e3
        print(f"  {e:2d} {names[e]:22s} {np.median(rel):8.2f}")
    per_tile = (t[:, 2:8, 0] - t[:, 1:7, 0]) / 1e3
    print(f"tile period (Q ready -> next Q ready): median {np.median(per_tile):.2f} us")
    s = t[:, ks, 1:9].astype(np.float64)
    dpair = np.diff(s, axis=2) / 1e3
    print(f"pair period (S ready spacing, pairs 1-7): median {np.median(dpair[dpair > 0]):.2f} us")
    gap = (t[:, 2:8, 1] - t[:, 1:7, 24]) / 1e3
    print(f"tile k done -> tile k+1 S ready pair 0: median {np.median(gap):.2f} us")


if __name__ == "__main__":
    main()
