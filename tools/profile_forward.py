"""Profiling target (analysis only): a few SLA2 forwards at a bench config, nothing else.

  ncu --set full -k regex:sla2_sparse_bf16 --launch-skip 2 -c 1 -o gpurun_out/sparse \\
      python tools/profile_forward.py --config cfg2
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
      python tools/profile_forward.py --config cfg2 --iters 2

Inputs are seeded randn (bf16) of the bench shape; --quant selects the INT8 QAT path."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {"cfg1": (1, 2, 4096), "cfg2": (1, 12, 32760), "cfg2pad": (1, 12, 32768), "cfg3": (1, 12, 75600), "cfg4": (1, 40, 75600)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--k-percent", type=float, default=3.0)
    ap.add_argument("--quant", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2602_12675_b200 as sla2
    B, H, N = CONFIGS[a.config]
    d = 128
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((B, H, N, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    eye = torch.eye(d, device=dev)[None]
    pq = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    pk = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    rho = torch.zeros((H, -(-N // 128)), device=dev)
    for _ in range(a.iters):
        sla2.forward(q, k, v, pq, pk, rho, k_percent=a.k_percent, quant=a.quant)
    torch.cuda.synchronize()
    print("ok", a.config, a.iters)


if __name__ == "__main__":
    main()
