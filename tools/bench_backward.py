"""Backward timing (analysis; the bench.py contract covers the forward): one SLA2 backward
(sla2_backward, hard routing, fp32 CUDA cores) at the fp32 config-1 geometry scaled up, and the
reference's own sla2_backward on one head on the host for context. Prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2602_12675_b200 as sla2  # noqa: E402


def main():
    B, H, N = 1, 2, int(os.environ.get("N", "4096"))
    d, bq, bk = int(os.environ.get("D", "64")), int(os.environ.get("BQ", "64")), int(os.environ.get("BK", "64"))
    kp = float(os.environ.get("KP", "10.0"))
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, dout = (torch.randn((B, H, N, d), generator=g, device=dev) for _ in range(4))
    eye = torch.eye(d, device=dev)[None]
    pq = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    pk = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    rho = torch.rand((H, N // bq), generator=g, device=dev) * 2 - 1
    out, mask, sv = sla2.forward(q, k, v, pq, pk, rho, k_percent=kp, bq=bq, bk=bk, return_mask=True, saved=True)
    for _ in range(3):
        sla2.sla2_backward(q, k, v, dout, rho, mask, sv, bq=bq, bk=bk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sla2.sla2_backward(q, k, v, dout, rho, mask, sv, bq=bq, bk=bk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    ref_ms = None
    try:
        import oracle_ctypes as oc
        R = oc.ref()
        if R is not None:
            os.environ["SLA2_THREADS"] = str(os.cpu_count() or 1)
            h = 0
            args = [x.cpu().numpy()[0, h] for x in (q, k, v)]
            t0 = time.perf_counter()
            R.backward(*args, bq, bk, mask.cpu().numpy()[0, h], rho.cpu().numpy()[h], dout.cpu().numpy()[0, h])
            ref_ms = (time.perf_counter() - t0) * 1e3 * B * H  # forward + backward, extrapolated
    except Exception as ex:  # context only
        ref_ms = f"unavailable: {ex}"
    print(json.dumps({"what": "sla2_backward (hard routing, fp32)", "B": B, "H": H, "N": N, "d": d, "bq": bq,
                      "bk": bk, "k_percent": kp, "device_ms": ms,
                      "reference_cpu_fwd_plus_bwd_ms": ref_ms, "cpu_threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
