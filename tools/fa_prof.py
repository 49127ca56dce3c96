"""Times the split forward's kernels at cfg2 (analysis helper): sparse forward stages, dense
full_attention, each with CUDA events; with NCU=1 runs one forward + one dense call only."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_12675_b200 as sla2
from paper_2602_12675_b200 import dist as sd

dev = torch.device("cuda:0")
H, N, d = 12, 32760, 128
tm = -(-N // 128)
q, k, v, pq, pk, rho = sd.shard_inputs(0, H, 1, N, d, tm, torch.bfloat16, dev, 1234)
if os.environ.get("NCU"):
    sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)
    sla2.full_attention(q[:, :2], k[:, :2], v[:, :2])
    torch.cuda.synchronize()
    sys.exit(0)


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("forward ms", timeit(lambda: sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)))
sla2.enable_stage_timing(True)
sla2.forward(q, k, v, pq, pk, rho, k_percent=3.0)
print("stages", sla2.last_stage_ms(timeline=True))
sla2.enable_stage_timing(False)
dms = timeit(lambda: sla2.full_attention(q, k, v), 3)
print(f"dense ms {dms:.3f}  TFLOPS {4 * N * N * d * H / dms / 1e9:.1f}")
