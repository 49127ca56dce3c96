"""Analysis only: sla2_forward_host wall time at cfg2 (pinned host buffers), for A/B runs."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2602_12675_b200 as sla2  # noqa: E402

B, H, N, d = 1, 12, 32760, 128
g = torch.Generator().manual_seed(0)
hq, hk, hv = (torch.randn((B, H, N, d), generator=g).to(torch.bfloat16).pin_memory() for _ in range(3))
eye = torch.eye(d)[None]
hpq = (eye + 0.05 * torch.randn((H, d, d), generator=g)).contiguous().pin_memory()
hpk = (eye + 0.05 * torch.randn((H, d, d), generator=g)).contiguous().pin_memory()
hrho = torch.zeros((H, -(-N // 128))).pin_memory()
hout = torch.empty_like(hq).pin_memory()
cp = sla2.FwdParams(B, H, N, d).c()
L = sla2.lib()
for _ in range(3):
    assert L.sla2_forward_host(C.byref(cp), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), hpq.data_ptr(),
                               hpk.data_ptr(), hrho.data_ptr(), hout.data_ptr(), None) == 0
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    L.sla2_forward_host(C.byref(cp), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), hpq.data_ptr(), hpk.data_ptr(),
                        hrho.data_ptr(), hout.data_ptr(), None)
    ts.append(time.perf_counter() - t0)
ts.sort()
x = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
bw = 5 * (256 << 20) / (time.perf_counter() - t0) / 1e9
print(f"SLA2_H2D_STREAMS={os.environ.get('SLA2_H2D_STREAMS', '2')}: median {ts[5] * 1e3:.3f} ms, best {ts[0] * 1e3:.3f} ms;"
      f" plain pinned H2D {bw:.1f} GB/s")
