"""Forward time and stage split at a chosen shape (analysis helper): H, N, KP env (default cfg4)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_12675_b200 as sla2
from paper_2602_12675_b200 import dist as sd

dev = torch.device("cuda:0")
H, N, d = int(os.environ.get("H", "40")), int(os.environ.get("N", "75600")), 128
kp = float(os.environ.get("KP", "3.0"))
tm = -(-N // 128)
q, k, v, pq, pk, rho = sd.shard_inputs(0, H, 1, N, d, tm, torch.bfloat16, dev, 1234)
fn = lambda: sla2.forward(q, k, v, pq, pk, rho, k_percent=kp)
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    fn()
e1.record()
torch.cuda.synchronize()
sla2.enable_stage_timing(True)
fn()
st = sla2.last_stage_ms(timeline=True)
sla2.enable_stage_timing(False)
print(f"H{H} N{N}: forward {e0.elapsed_time(e1) / 5:.3f} ms  router {st[0]:.3f}  sparse {st[2]:.3f}  "
      f"timeline mu {st[4]:.3f} keyprep {st[6]:.3f} router_back {st[7]:.3f} lin {st[8]:.3f}")
