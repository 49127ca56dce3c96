"""Parity of the sm_100a SLA2 forward (through the C ABI) against the CPU oracle.

Bar (north star): router mask bits and kept-block index lists bit-exact; outputs within
1e-2 normwise relative for bf16 (max|gpu-ref| <= 1e-2 * max|ref|) and max-abs 1e-4 for fp32,
the reference's own float tolerance (test_attention.cpp:232-241)."""
import numpy as np
import pytest

import paper_2602_12675_b200 as sla2
from sla2_testlib import (make_inputs, mask_to_idx, oracle_head, oracle_router_head, rel_err, to_dev)

pytestmark = pytest.mark.gpu

BF16_TOL = 1e-2
F32_TOL = 1e-4


def _torch():
    import torch
    return torch


# ----------------------------------------------------------------------------- router
@pytest.mark.parametrize("N,k_percent,sigma,seed", [(4096, 3.0, 1.0, 1), (8192, 3.0, 1.0, 2), (8192, 10.0, 4.0, 3),
                                                   (16384, 5.0, 1.0, 4),
                                                   (16384, 30.0, 1.0, 8),    # kappa 77: bitonic top-k
                                                   (65536, 3.0, 1.0, 9),     # tn 1024: 64-key register top-k
                                                   (32768, 3.0, 1.0, 10)])   # the cfg2 geometry
def test_router_bitexact_bf16(cuda, N, k_percent, sigma, seed):
    torch = _torch()
    B, H, d, bq, bk = 1, 3, 128, 128, 64
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, seed, sigma)
    pc, mask, idx = sla2.router(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                to_dev(pq, torch.float32, cuda), to_dev(pk, torch.float32, cuda),
                                k_percent=k_percent, bq=bq, bk=bk)
    pc, mask, idx = pc.cpu().numpy(), mask.cpu().numpy(), idx.cpu().numpy()
    for h in range(H):
        rpc, rmask, kappa = oracle_router_head(q[0, h], k[0, h], pq[h], pk[h], bq, bk, k_percent)
        assert np.array_equal(pc[0, h].view(np.uint32), rpc.view(np.uint32)), f"pc bits differ (head {h})"
        assert np.array_equal(mask[0, h], rmask), f"mask differs (head {h})"
        ridx = np.stack(mask_to_idx(rmask))
        assert ridx.shape[1] == kappa
        assert np.array_equal(idx[0, h], ridx)


@pytest.mark.gpu
@pytest.mark.parametrize("k_percent", [3.0, 30.0, 60.0])
def test_router_topk_ties_and_paths(cuda, k_percent):
    """The router's top-k paths (candidate bound with 1 or 2 minima per lane, the radix
    fallback on overflow, kappa > 64) on rows with exact ties: zero query blocks give uniform
    rows (every key equal), duplicated key blocks give equal scores inside a row."""
    torch = _torch()
    B, H, N, d, bq, bk = 1, 2, 8192, 128, 128, 64
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 77)
    q[:, :, : 4 * bq] = 0.0
    k[:, :, 9 * bk: 10 * bk] = k[:, :, 5 * bk: 6 * bk]
    k[:, :, 20 * bk: 21 * bk] = k[:, :, 5 * bk: 6 * bk]
    pc, mask, idx = sla2.router(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                to_dev(pq, torch.float32, cuda), to_dev(pk, torch.float32, cuda),
                                k_percent=k_percent, bq=bq, bk=bk)
    for h in range(H):
        rpc, rmask, kappa = oracle_router_head(q[0, h], k[0, h], pq[h], pk[h], bq, bk, k_percent)
        assert np.array_equal(pc.cpu().numpy()[0, h].view(np.uint32), rpc.view(np.uint32))
        assert np.array_equal(mask.cpu().numpy()[0, h], rmask), (h, kappa)
        assert np.array_equal(idx.cpu().numpy()[0, h], np.stack(mask_to_idx(rmask)))


@pytest.mark.gpu
def test_router_bitexact_f32_cfg1(cuda):
    torch = _torch()
    B, H, N, d, bq, bk, kp = 1, 2, 4096, 64, 64, 64, 10.0
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 11, 1.0, bf16=False, bq=bq, bk=bk)
    pc, mask, idx = sla2.router(to_dev(q, torch.float32, cuda), to_dev(k, torch.float32, cuda),
                                to_dev(pq, torch.float32, cuda), to_dev(pk, torch.float32, cuda), k_percent=kp,
                                bq=bq, bk=bk)
    for h in range(H):
        rpc, rmask, kappa = oracle_router_head(q[0, h], k[0, h], pq[h], pk[h], bq, bk, kp)
        assert np.array_equal(pc.cpu().numpy()[0, h].view(np.uint32), rpc.view(np.uint32))
        assert np.array_equal(mask.cpu().numpy()[0, h], rmask)
        assert np.array_equal(idx.cpu().numpy()[0, h], np.stack(mask_to_idx(rmask)))


# ----------------------------------------------------------------------------- bf16 forward
@pytest.mark.parametrize("N,H,k_percent,seed", [(4096, 2, 3.0, 5), (8192, 2, 10.0, 6), (2048, 1, 50.0, 7)])
def test_forward_bf16_vs_oracle(cuda, N, H, k_percent, seed):
    torch = _torch()
    B, d, bq, bk = 1, 128, 128, 64
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, seed)
    out, mask, sv = sla2.forward(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                 to_dev(v, torch.bfloat16, cuda), to_dev(pq, torch.float32, cuda),
                                 to_dev(pk, torch.float32, cuda), to_dev(rho, torch.float32, cuda),
                                 k_percent=k_percent, return_mask=True, saved=True)
    out = out.float().cpu().numpy()
    for h in range(H):
        r_out, r_mask, r_os, r_ol, r_l = oracle_head(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], bq, bk,
                                                     k_percent)
        assert np.array_equal(mask.cpu().numpy()[0, h], r_mask)
        e_max, e_l2 = rel_err(out[0, h], r_out)
        assert e_max <= BF16_TOL, (h, e_max, e_l2)
        e_os = rel_err(sv["o_s"].cpu().numpy()[0, h], r_os)
        e_ol = rel_err(sv["o_l"].cpu().numpy()[0, h], r_ol)
        assert e_os[0] <= BF16_TOL, ("o_s", e_os)
        assert e_ol[0] <= BF16_TOL, ("o_l", e_ol)
        np.testing.assert_allclose(sv["big_l"].cpu().numpy()[0, h], r_l, atol=2e-2, rtol=2e-3)


def test_forward_bf16_batch_layout(cuda):
    """B > 1 with per-head router state shared across the batch (model.hpp:38-39)."""
    torch = _torch()
    B, H, N, d = 2, 2, 2048, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 21)
    out = sla2.forward(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                       to_dev(v, torch.bfloat16, cuda), to_dev(pq, torch.float32, cuda),
                       to_dev(pk, torch.float32, cuda), to_dev(rho, torch.float32, cuda), k_percent=5.0)
    out = out.float().cpu().numpy()
    for b in range(B):
        for h in range(H):
            r = oracle_head(q[b, h], k[b, h], v[b, h], pq[h], pk[h], rho[h], 128, 64, 5.0)[0]
            assert rel_err(out[b, h], r)[0] <= BF16_TOL


@pytest.mark.parametrize("quant", [False, True])
def test_forward_host_matches_device(cuda, quant):
    """sla2_forward_host (host buffers, per-head copy/compute pipeline) returns exactly what
    one device-side sla2_forward over all heads returns, mask included."""
    torch = _torch()
    B, H, N, d = 2, 3, 4096, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 22)
    hq, hk, hv = (torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in (q, k, v))
    hpq, hpk, hrho = (torch.from_numpy(x) for x in (pq, pk, rho))
    out_h, mask_h = sla2.forward_host(hq, hk, hv, hpq, hpk, hrho, k_percent=3.0, quant=quant, return_mask=True)
    out_d, mask_d = sla2.forward(hq.to(cuda), hk.to(cuda), hv.to(cuda), hpq.to(cuda), hpk.to(cuda), hrho.to(cuda),
                                 k_percent=3.0, quant=quant, return_mask=True)
    assert torch.equal(mask_h, mask_d.cpu())
    assert torch.equal(out_h, out_d.cpu())
    r = oracle_head(q[1, 2], k[1, 2], v[1, 2], pq[2], pk[2], rho[2], 128, 64, 3.0, quant=quant)[0]
    assert rel_err(out_h.float().numpy()[1, 2], r)[0] <= BF16_TOL


def test_captured_forward_matches_eager(cuda):
    """CapturedForward (the forward as one CUDA graph) replays to exactly the eager result,
    and picks up new inputs written into the captured tensors."""
    torch = _torch()
    B, H, N, d = 1, 2, 4096, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 23)
    dev = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    eager = sla2.forward(*dev, k_percent=3.0).clone()
    g = sla2.CapturedForward(*dev, k_percent=3.0)
    assert torch.equal(g(), eager)
    q2, k2, v2 = make_inputs(B, H, N, d, 24)[:3]
    for t, x in zip(dev[:3], (q2, k2, v2)):
        t.copy_(to_dev(x, torch.bfloat16, cuda))
    assert torch.equal(g(), sla2.forward(*dev, k_percent=3.0))


# ----------------------------------------------------------------------------- INT8 QAT forward
@pytest.mark.parametrize("N,H,k_percent,seed", [(4096, 2, 3.0, 51), (8192, 1, 10.0, 52), (2048, 1, 100.0, 53)])
def test_forward_qat_vs_oracle(cuda, N, H, k_percent, seed):
    """QuantConfig INT8 on QK and PV (quant.hpp:15-19): codes, scales and S are the
    reference's; output within the low-bit tolerance of the oracle's QAT forward."""
    torch = _torch()
    B, d, bq, bk = 1, 128, 128, 64
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, seed)
    out, mask, sv = sla2.forward(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                 to_dev(v, torch.bfloat16, cuda), to_dev(pq, torch.float32, cuda),
                                 to_dev(pk, torch.float32, cuda), to_dev(rho, torch.float32, cuda),
                                 k_percent=k_percent, quant=True, return_mask=True, saved=True)
    out = out.float().cpu().numpy()
    for h in range(H):
        r_out, r_mask, r_os, r_ol, r_l = oracle_head(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], bq, bk,
                                                     k_percent, quant=True)
        assert np.array_equal(mask.cpu().numpy()[0, h], r_mask)
        assert rel_err(out[0, h], r_out)[0] <= BF16_TOL
        assert rel_err(sv["o_s"].cpu().numpy()[0, h], r_os)[0] <= BF16_TOL
        np.testing.assert_allclose(sv["big_l"].cpu().numpy()[0, h], r_l, atol=1e-3, rtol=1e-4)


# ----------------------------------------------------------------------------- fp32 forward
@pytest.mark.parametrize("N,d,bq,bk,k_percent", [(4096, 64, 64, 64, 10.0), (1024, 32, 32, 16, 25.0),
                                                 (64, 8, 8, 4, 10.0), (64, 8, 8, 4, 50.0),
                                                 (32, 8, 4, 4, 25.0), (32, 8, 4, 8, 25.0),   # bq < 8
                                                 (2048, 128, 128, 64, 5.0),                  # Wan blocks, fp32
                                                 (1024, 64, 256, 64, 25.0)])                 # bq 256: 1 thread/row
def test_forward_f32_vs_oracle(cuda, N, d, bq, bk, k_percent):
    torch = _torch()
    B, H = 1, 2
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 31, bf16=False, bq=bq, bk=bk)
    out, mask = sla2.forward(to_dev(q, torch.float32, cuda), to_dev(k, torch.float32, cuda),
                             to_dev(v, torch.float32, cuda), to_dev(pq, torch.float32, cuda),
                             to_dev(pk, torch.float32, cuda), to_dev(rho, torch.float32, cuda),
                             k_percent=k_percent, bq=bq, bk=bk, return_mask=True)
    for h in range(H):
        r_out, r_mask = oracle_head(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], bq, bk, k_percent)[:2]
        assert np.array_equal(mask.cpu().numpy()[0, h], r_mask)
        assert np.abs(out.cpu().numpy()[0, h] - r_out).max() <= F32_TOL


# ----------------------------------------------------------------------------- blockwise with masks
def test_full_mask_is_full_attention(cuda):
    """BlockMask::ones: alpha forced to 1, equals full attention (test_attention.cpp:167-174)."""
    torch = _torch()
    B, H, N, d = 1, 2, 2048, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 41)
    qd, kd, vd = (to_dev(x, torch.bfloat16, cuda) for x in (q, k, v))
    mask = torch.ones((B, H, N // 128, N // 64), dtype=torch.uint8, device=cuda)
    out = sla2.sla2_forward_blockwise(qd, kd, vd, mask, to_dev(rho, torch.float32, cuda))
    ref = torch.nn.functional.scaled_dot_product_attention(qd.float(), kd.float(), vd.float())
    assert rel_err(out.float().cpu().numpy(), ref.cpu().numpy())[0] <= BF16_TOL
    dense = sla2.full_attention(qd, kd, vd)
    assert rel_err(dense.float().cpu().numpy(), ref.cpu().numpy())[0] <= BF16_TOL


def test_ragged_mask_rows(cuda):
    """Random masks with different kept counts per row (random_mask, test_attention.cpp:40-42)."""
    torch = _torch()
    import oracle_ctypes as oc
    B, H, N, d = 1, 1, 2048, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 43)
    rng = np.random.default_rng(0)
    tm, tn = N // 128, N // 64
    m = (rng.random((tm, tn)) < 0.1).astype(np.uint8)
    m[np.arange(tm), rng.integers(0, tn, tm)] = 1
    m[3, :] = 1  # one full row
    out = sla2.sla2_forward_blockwise(*(to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)),
                                      torch.from_numpy(m[None, None]).to(cuda), to_dev(rho, torch.float32, cuda))
    r = oc.port().forward_blockwise(q[0, 0], k[0, 0], v[0, 0], 128, 64, m, rho[0])[0]
    assert rel_err(out.float().cpu().numpy()[0, 0], r)[0] <= BF16_TOL


def test_empty_mask_row_raises(cuda):
    """attention.hpp:442-447 / test_attention.cpp:305-311."""
    torch = _torch()
    B, H, N, d = 1, 1, 1024, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 44)
    mask = torch.ones((1, 1, N // 128, N // 64), dtype=torch.uint8, device=cuda)
    mask[0, 0, 2] = 0
    with pytest.raises(sla2.ShapeError):
        sla2.sla2_forward_blockwise(*(to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)), mask,
                                    to_dev(rho, torch.float32, cuda))


def test_budget_edges(cuda):
    """kappa = 1 (tiny k%) and kappa = tn (k = 100: every row full, alpha forced to 1)."""
    torch = _torch()
    B, H, N, d = 1, 1, 2048, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 45)
    dev = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    for kp in (0.01, 100.0):
        out, mask = sla2.forward(*dev, k_percent=kp, return_mask=True)
        r_out, r_mask = oracle_head(q[0, 0], k[0, 0], v[0, 0], pq[0], pk[0], rho[0], 128, 64, kp)[:2]
        assert np.array_equal(mask.cpu().numpy()[0, 0], r_mask)
        assert rel_err(out.float().cpu().numpy()[0, 0], r_out)[0] <= BF16_TOL


def test_deterministic(cuda):
    torch = _torch()
    B, H, N, d = 1, 2, 4096, 128
    q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 46)
    dev = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    a = sla2.forward(*dev).clone()
    b = sla2.forward(*dev)
    assert torch.equal(a, b)


# ----------------------------------------------------------------------------- reference goldens
def _goldens():
    import os
    g = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return sorted(os.path.join(g, f) for f in os.listdir(g) if f.endswith(".npz") and not f.startswith(("backward_", "soft_")))


@pytest.mark.parametrize("path", _goldens(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_gpu_vs_reference_golden(cuda, path):
    """GPU path against outputs of the unmodified reference (tests/golden/make_golden.py)."""
    torch = _torch()
    g = np.load(path)
    q, k, v = g["q"], g["k"], g["v"]
    if q.dtype != np.float32:
        pytest.skip("double-precision reference case (no fp64 GPU path)")
    bq, bk, kp, quant = int(g["bq"]), int(g["bk"]), float(g["k_percent"]), bool(g["quant"])
    bf16 = (q.shape[1] == 128 and bq == 128 and bk == 64)
    if quant and not bf16:
        pytest.skip("QAT runs on the bf16 kernel geometry")
    dt = torch.bfloat16 if bf16 else torch.float32
    dev = [to_dev(x[None, None], dt, cuda) for x in (q, k, v)]
    dev += [to_dev(g["proj_q"][None], torch.float32, cuda), to_dev(g["proj_k"][None], torch.float32, cuda),
            to_dev(g["rho"][None], torch.float32, cuda)]
    try:
        out, mask = sla2.forward(*dev, k_percent=kp, bq=bq, bk=bk, quant=quant, return_mask=True)
    except sla2.ContractError as e:
        pytest.skip(str(e))
    assert np.array_equal(mask.cpu().numpy()[0, 0], g["mask"])
    got = out.float().cpu().numpy()[0, 0]
    if bf16:
        assert rel_err(got, g["out"])[0] <= BF16_TOL
    else:
        assert np.abs(got - g["out"]).max() <= F32_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,N", [(1, 2, 2048),   # tm even: the two lanes share one K / V ring
                                   (1, 3, 1920),   # tm odd: independent lanes
                                   (2, 1, 1000),   # ragged N (partial last query and key blocks)
                                   (1, 1, 130),    # fewer query blocks than lanes on one SM
                                   (1, 5, 640)])   # more CTAs' worth of lanes than query blocks per head
def test_dense_attention_kernel_vs_sdpa(cuda, B, H, N):
    """full_attention (attention.hpp:71-75) on the two-query-block tcgen05 kernel (sparse_fa.cu,
    dense mode) against fp32 SDPA on the same bf16 inputs: within 1e-2 normwise."""
    import torch
    g = torch.Generator(device=cuda).manual_seed(N + H)
    q, k, v = (torch.randn((B, H, N, 128), generator=g, device=cuda).to(torch.bfloat16) for _ in range(3))
    o = sla2.full_attention(q, k, v).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float())
    assert ((o - ref).abs().max() / ref.abs().max()).item() <= 1e-2
