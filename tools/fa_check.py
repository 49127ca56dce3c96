"""sparse_fa.cu check on the GPU (analysis helper): the split forward (linear-branch kernel +
two-query-block attention kernel) vs the saved-state path (sparse_bf16.cu) and the oracle, and
the dense mode vs torch SDPA (fp32)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import paper_2602_12675_b200 as sla2
from sla2_testlib import make_inputs, oracle_head, rel_err, to_dev

dev = torch.device("cuda:0")
cases = [(1, 1, 2048, 5.0), (2, 2, 2048, 5.0), (1, 2, 4096, 3.0), (1, 3, 8192, 10.0), (1, 12, 32768, 3.0),
         (1, 2, 32760, 3.0), (1, 1, 8200, 100.0), (1, 2, 4096, 50.0), (1, 1, 1000, 30.0), (1, 3, 130, 50.0)]
for B, H, N, kp in cases:
    q, k, v, pq, pk, rho = make_inputs(B, H, -(-N // 128) * 128, 128, seed=N + H)
    q, k, v = (np.ascontiguousarray(x[:, :, :N]) for x in (q, k, v))
    d = [to_dev(x, torch.bfloat16, dev) for x in (q, k, v)] + [to_dev(x, torch.float32, dev) for x in (pq, pk, rho)]
    t0 = time.time()
    o2 = sla2.forward(*d, k_percent=kp)
    torch.cuda.synchronize()
    o1, sv = sla2.forward(*d, k_percent=kp, saved=True)
    torch.cuda.synchronize()
    e = rel_err(o2.float().cpu().numpy(), o1.float().cpu().numpy())
    line = f"B{B} H{H} N{N} k{kp}: fa vs v1 {e[0]:.2e}"
    if N % 128 == 0 and N <= 8192:
        r = oracle_head(q[0, 0], k[0, 0], v[0, 0], pq[0], pk[0], rho[0], 128, 64, kp)[0]
        line += f"  fa vs oracle {rel_err(o2[0, 0].float().cpu().numpy(), r)[0]:.2e}"
    print(line, f"({time.time() - t0:.1f}s)", flush=True)
for B, H, N in [(1, 2, 1024), (1, 2, 4096), (2, 3, 2000), (1, 1, 130)]:
    g = torch.Generator(device=dev).manual_seed(N)
    q, k, v = (torch.randn((B, H, N, 128), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    o = sla2.full_attention(q, k, v).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
    err = ((o - ref).abs().max() / ref.abs().max()).item()
    print(f"dense B{B} H{H} N{N}: vs sdpa fp32 {err:.2e}", flush=True)
