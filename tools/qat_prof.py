"""QAT forward at cfg3 (analysis helper): the two-lane INT8 kernel path vs the saved-state path
(sla2_sparse_i8_kernel) on the same inputs, and the forward time; NCU=1 runs one forward only."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_12675_b200 as sla2
from paper_2602_12675_b200 import dist as sd

dev = torch.device("cuda:0")
H, N, d = int(os.environ.get("H", "12")), 32768, 128
tm = N // 128
q, k, v, pq, pk, rho = sd.shard_inputs(0, H, 1, N, d, tm, torch.bfloat16, dev, 1234)
if os.environ.get("NCU"):
    sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True)
    torch.cuda.synchronize()
    sys.exit(0)
o_new = sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True).float()
o_old, _ = sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True, saved=True)
o_old = o_old.float()
print("new vs saved-path kernel: max|d| / max|ref| =", ((o_new - o_old).abs().max() / o_old.abs().max()).item())
for _ in range(3):
    sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0, quant=True)
e1.record()
torch.cuda.synchronize()
print("qat forward ms", e0.elapsed_time(e1) / 10)
