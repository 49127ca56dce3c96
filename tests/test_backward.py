"""SLA2 backward, hard routing (attention.hpp:610-809): the device
sla2_backward against the UNMODIFIED reference's own sla2_backward (oracle/_ref, which travels
to the GPU box prebuilt) on identical inputs, mask and upstream gradient. fp32 (the backward is
full precision); tolerance 1e-4 normwise (max|gpu - ref| <= 1e-4 max|ref|), the
reference's float tolerance (test_attention.cpp:232-241). The forward state the device
backward consumes (O_s, O_l, L) comes from the device forward."""
import numpy as np
import pytest

import oracle_ctypes as oc
import paper_2602_12675_b200 as sla2

R = oc.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built (no /root/reference here)")
TOL = 1e-4


def _rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@needs_ref
def test_reference_backward_binding_cpu():
    """The reference backward runs through the shim and its dv matches a dense restatement of
    the sparse branch's dV on a full mask with alpha forced to 1 (no linear branch)."""
    P = oc.port()
    n, d, bq, bk = 32, 8, 8, 8
    q, k, v = (P.gaussian((n, d), 700 + i) for i in range(3))
    d_out = P.gaussian((n, d), 710)
    mask = np.ones((n // bq, n // bk), np.uint8)
    dq, dk, dv, drho, o_s, o_l, big_l = R.backward(q, k, v, bq, bk, mask, np.zeros(n // bq), d_out)
    kt = k - k.mean(axis=0)
    s = q @ kt.T / np.sqrt(d)
    p = np.exp(s - s.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    assert np.abs(dv - p.T @ d_out).max() <= 1e-10
    assert np.all(drho == 0.0)  # full rows: alpha is forced to 1


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("N,H,d,bq,bk,kp,smooth,seed", [(1024, 2, 64, 64, 64, 25.0, True, 1),
                                                         (512, 1, 64, 32, 64, 10.0, True, 2),
                                                         (512, 1, 32, 64, 32, 30.0, False, 3),
                                                         (256, 1, 64, 64, 64, 100.0, True, 4),
                                                         # the Wan2.1 block shape (d = 128, bq = 128, bk = 64)
                                                         (1024, 1, 128, 128, 64, 10.0, True, 5),
                                                         (512, 2, 128, 128, 64, 25.0, False, 6),
                                                         (512, 1, 96, 64, 32, 20.0, True, 7)])
def test_backward_vs_reference(cuda, N, H, d, bq, bk, kp, smooth, seed):
    import torch
    from sla2_testlib import make_inputs, to_dev
    q, k, v, pq, pk, rho = make_inputs(1, H, N, d, seed, bf16=False, bq=bq, bk=bk)
    d_out = np.random.default_rng(seed + 100).standard_normal((1, H, N, d)).astype(np.float32)
    dev = [to_dev(x, torch.float32, cuda) for x in (q, k, v, pq, pk, rho)]
    out, mask, sv = sla2.forward(*dev, k_percent=kp, bq=bq, bk=bk, smooth=smooth, return_mask=True, saved=True)
    g = sla2.sla2_backward(dev[0], dev[1], dev[2], to_dev(d_out, torch.float32, cuda), dev[5], mask, sv, bq=bq, bk=bk,
                           smooth=smooth)
    mask = mask.cpu().numpy()
    for h in range(H):
        rdq, rdk, rdv, rdrho = R.backward(q[0, h], k[0, h], v[0, h], bq, bk, mask[0, h], rho[h], d_out[0, h],
                                          smooth=smooth)[:4]
        assert _rel(g["dq"].cpu().numpy()[0, h], rdq) <= TOL, ("dq", h)
        assert _rel(g["dk"].cpu().numpy()[0, h], rdk) <= TOL, ("dk", h)
        assert _rel(g["dv"].cpu().numpy()[0, h], rdv) <= TOL, ("dv", h)
        if np.abs(rdrho).max() > 0:
            assert _rel(g["drho"].cpu().numpy()[0, h], rdrho) <= TOL, ("drho", h)
        else:
            assert np.all(g["drho"].cpu().numpy()[0, h] == 0)


@pytest.mark.gpu
def test_backward_contract(cuda):
    import torch
    x = torch.zeros((1, 1, 512, 256), device=cuda)
    m = torch.ones((1, 1, 8, 8), dtype=torch.uint8, device=cuda)
    with pytest.raises(sla2.ContractError):  # d = 256 > 128 on this path
        sla2.sla2_backward(x, x, x, x, torch.zeros((1, 8), device=cuda), m,
                           {"o_s": x, "o_l": x, "big_l": x[..., 0].contiguous()}, bq=64, bk=64)
    x = torch.zeros((1, 1, 512, 128), device=cuda)
    m = torch.ones((1, 1, 2, 4), dtype=torch.uint8, device=cuda)
    with pytest.raises(sla2.ContractError):  # bq = 256 > 128 with d > 64
        sla2.sla2_backward(x, x, x, x, torch.zeros((1, 2), device=cuda), m,
                           {"o_s": x, "o_l": x, "big_l": x[..., 0].contiguous()}, bq=256, bk=128)


def _bwd_goldens():
    import os
    g = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return sorted(os.path.join(g, f) for f in os.listdir(g) if f.startswith("backward_") and f.endswith(".npz"))


@pytest.mark.gpu
@pytest.mark.parametrize("path", _bwd_goldens(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_backward_vs_reference_golden(cuda, path):
    """The same check against fixtures the reference wrote (tests/golden/make_backward_golden.py):
    no oracle/_ref needed."""
    import torch
    z = np.load(path)
    bq, bk = int(z["bq"]), int(z["bk"])
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x))[None, None].to(cuda)  # noqa: E731
    q, k, v, d_out = t(z["q"]), t(z["k"]), t(z["v"]), t(z["d_out"])
    pq, pk = (torch.from_numpy(z[n])[None].to(cuda) for n in ("proj_q", "proj_k"))
    rho = torch.from_numpy(z["rho"])[None].to(cuda)
    out, mask, sv = sla2.forward(q, k, v, pq, pk, rho, k_percent=float(z["k_percent"]), bq=bq, bk=bk,
                                 return_mask=True, saved=True)
    assert np.array_equal(mask.cpu().numpy()[0, 0], z["mask"])
    g = sla2.sla2_backward(q, k, v, d_out, rho, mask, sv, bq=bq, bk=bk)
    for name in ("dq", "dk", "dv"):
        assert _rel(g[name].cpu().numpy()[0, 0], z[name]) <= TOL, name
    assert _rel(g["drho"].cpu().numpy()[0, 0], z["drho"]) <= TOL
