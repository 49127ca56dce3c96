"""Parity at the BENCHMARKED configurations (BASELINE.json configs[1..4]) and of the whole saved
state, through the C ABI, against the unmodified reference (oracle/_ref) wherever the reference
accepts the shape, else against the C port's ragged extension (pinned to the reference on
divisible N, tests/test_ragged.py).

Bars: every head's mask and kept-block index list bit-exact; two sampled heads' outputs within
1e-2 normwise (max|gpu - ref| <= 1e-2 * max|ref|, per branch); the QAT operand codes and scales
(quantize, quant.hpp:31-50) and the dequantized QAT scores S (block_scores_qk, attention.hpp:
372-394) bit-exact."""
import os

import numpy as np
import pytest

import oracle_ctypes as oc
import paper_2602_12675_b200 as sla2
from sla2_testlib import (make_inputs, mask_to_idx, oracle_attention_any, oracle_router_any, rel_err, to_dev)

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _threads():
    n = os.cpu_count() or 1
    os.environ.setdefault("SLA2_THREADS", str(n))  # the reference reads it once (common.hpp:31-43)
    oc.port()._set_threads(n)


def _inputs(B, H, N, seed):
    """Seeded inputs at any N (ragged N: the block-multiple draw truncated to N rows)."""
    npad = -(-N // 128) * 128
    q, k, v, pq, pk, _ = make_inputs(B, H, npad, 128, seed)
    q, k, v = (np.ascontiguousarray(x[:, :, :N]) for x in (q, k, v))
    rho = np.random.default_rng(seed + 1000).uniform(-1, 1, (H, -(-N // 128))).astype(np.float32)
    return q, k, v, pq, pk, rho


def _dev(cuda, q, k, v, pq, pk, rho):
    import torch
    return ([to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] +
            [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)])


def _check_full_call(cuda, N, H, seed, heads_out, quant=False, expect=None):
    """One sla2_forward over all H heads; every mask/idx vs the oracle router, `heads_out`
    output heads vs the oracle forward. Returns the oracle kinds used."""
    import torch
    _threads()
    B, kp = 1, 3.0
    q, k, v, pq, pk, rho = _inputs(B, H, N, seed)
    out, mask, idx, sv = sla2.forward(*_dev(cuda, q, k, v, pq, pk, rho), k_percent=kp, quant=quant,
                                      return_mask=True, return_idx=True, saved=True)
    torch.cuda.synchronize()
    mask, idx = mask.cpu().numpy(), idx.cpu().numpy()
    kinds = set()
    for h in range(H):
        _, rmask, kappa, which = oracle_router_any(q[0, h], k[0, h], pq[h], pk[h], 128, 64, kp)
        kinds.add(which)
        assert np.array_equal(mask[0, h], rmask), f"mask differs (head {h}, oracle {which})"
        assert np.array_equal(idx[0, h], np.stack(mask_to_idx(rmask))), f"kept-block list differs (head {h})"
    out = out.float().cpu().numpy()
    for h in heads_out:
        r_out, r_mask, r_os, r_ol, r_l, which = oracle_attention_any(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h],
                                                                     128, 64, kp, quant=quant)
        kinds.add(which)
        assert np.array_equal(mask[0, h], r_mask)
        assert rel_err(out[0, h], r_out)[0] <= TOL, (h, rel_err(out[0, h], r_out))
        assert rel_err(sv["o_s"][0, h].cpu().numpy(), r_os)[0] <= TOL
        if not r_mask.all():
            assert rel_err(sv["o_l"][0, h].cpu().numpy(), r_ol)[0] <= TOL
    assert np.isfinite(out).all()
    if expect:
        assert kinds == {expect}, kinds
    return q, k, v, pq, pk, rho


def test_cfg2_full_call_ragged(cuda):
    """BASELINE configs[1] as benchmarked: B=1, H=12, N=32760 (true Wan2.1-1.3B), 97%."""
    _check_full_call(cuda, 32760, 12, 101, heads_out=(0, 11), expect="port")


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
def test_cfg2_padded_full_call_reference(cuda):
    """The same at N=32768 (the reference's own shape rule), against the reference itself."""
    _check_full_call(cuda, 32768, 12, 102, heads_out=(0, 11), expect="reference")


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
def test_cfg3_qat_full_call_reference(cuda):
    """BASELINE configs[2]: INT8 QAT at B=1, H=12, N=32768: masks and 2 output heads vs the
    reference's QAT forward; every head's Q / K~ / V codes and scales bit-exact."""
    q, k, v, pq, pk, rho = _check_full_call(cuda, 32768, 12, 103, heads_out=(0, 11), quant=True, expect="reference")
    _check_codes(cuda, q, k, v, heads=range(12))


def test_cfg4_masks_ragged(cuda):
    """BASELINE configs[3]: B=1, H=40, N=75600 (Wan2.1-14B 720p): all 40 masks, 2 output heads."""
    _check_full_call(cuda, 75600, 40, 104, heads_out=(0, 39), expect="port")


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
def test_router_tn2048_kappa410_reference(cuda):
    """BASELINE configs[4]'s largest router: N=131072 (tn=2048) at 80% sparsity, kappa=410
    (router.hpp:36-40), against the reference's block_scores + hard_topk."""
    import torch
    _threads()
    N, H, kp = 131072, 2, 20.0
    q, k, v, pq, pk, rho = _inputs(1, H, N, 105)
    pc, mask, idx = sla2.router(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                to_dev(pq, torch.float32, cuda), to_dev(pk, torch.float32, cuda), k_percent=kp)
    assert idx.shape[-1] == 410
    for h in range(H):
        rpc, rmask, kappa, which = oracle_router_any(q[0, h], k[0, h], pq[h], pk[h], 128, 64, kp)
        assert which == "reference" and kappa == 410
        assert np.array_equal(pc[0, h].cpu().numpy().view(np.uint32), rpc.view(np.uint32)), h
        assert np.array_equal(mask[0, h].cpu().numpy(), rmask), h
        assert np.array_equal(idx[0, h].cpu().numpy(), np.stack(mask_to_idx(rmask))), h


# ----------------------------------------------------------------------------- QAT operands
def _check_codes(cuda, q, k, v, heads, bq=128, bk=64):
    """sla2_quantize (the kind::i8 kernel's operands) vs the reference's quantize per block."""
    import torch
    r = oc.ref()
    res = sla2.quantize(*(to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)))
    got = {n: t.cpu().numpy() for n, t in res.items()}
    N = q.shape[2]
    for h in heads:
        kt = r.smooth_k(k[0, h])[0]  # K~ = K - colmean(K) (quant.hpp:88-96)
        for which, x, blk, codes, scales in (("Q", q[0, h], bq, got["q_codes"], got["q_scales"]),
                                             ("K~", kt, bk, got["k_codes"], got["k_scales"]),
                                             ("V", v[0, h], bk, got["v_codes"], got["v_scales"])):
            for b in range(N // blk):
                rc, rs = r.quantize(x[b * blk:(b + 1) * blk])
                assert np.array_equal(codes[0, h, b * blk:(b + 1) * blk], rc), (which, h, b)
                assert np.float32(rs).view(np.uint32) == scales[0, h, b].view(np.uint32), (which, h, b)


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
def test_qat_codes_and_scales_bitexact(cuda):
    q, k, v, pq, pk, rho = _inputs(1, 2, 4096, 106)
    _check_codes(cuda, q, k, v, heads=range(2))


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("N", [4096, 32768])
def test_qat_scores_bitexact(cuda, N):
    """The i8 kernel's dequantized S (int32 tcgen05 accumulation, then fl(fl(acc * fl(sQ sK)) *
    1/sqrt d)) of each query block's first kept key block equals the reference's
    block_scores_qk with QuantConfig on the same blocks, bit for bit (sampled query blocks)."""
    import torch
    _threads()
    r = oc.ref()
    q, k, v, pq, pk, rho = _inputs(1, 1, N, 107)
    out, idx, sv = sla2.forward(*_dev(cuda, q, k, v, pq, pk, rho), k_percent=3.0, quant=True, return_idx=True,
                                saved="full")
    s_first = sv["qat_s_first"][0, 0].cpu().numpy()
    idx = idx[0, 0].cpu().numpy()
    kt = r.smooth_k(k[0, 0])[0]
    tm = N // 128
    for i in sorted(set(np.linspace(0, tm - 1, 12).astype(int))):
        j = int(idx[i, 0])
        ref_s = r.block_scores_qk(q[0, 0], kt, i * 128, 128, j * 64, 64, quant=True)
        assert np.array_equal(s_first[i].view(np.uint32), ref_s.view(np.uint32)), (i, j)


# ----------------------------------------------------------------------------- saved state
@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ["bf16", "qat", "f32"])
def test_saved_state_vs_reference(cuda, case):
    """SLA2ForwardSaved (attention.hpp:345-358) in full: q_phi / k_phi bit-exact (row_softmax in
    the reference's arithmetic), h_blocks / z_blocks (the per-query-block complements) within
    the branch tolerance (1e-2 bf16 / QAT, 1e-5 fp32), o_s / o_l / L as the forward tests."""
    import torch
    _threads()
    r = oc.ref()
    if case == "f32":
        N, d, bq, bk, kp, dt, tol = 1024, 64, 64, 64, 25.0, torch.float32, 1e-5
        q, k, v, pq, pk, rho = make_inputs(1, 1, N, d, 108, bf16=False, bq=bq, bk=bk)
    else:
        N, d, bq, bk, kp, dt, tol = 2048, 128, 128, 64, 10.0, torch.bfloat16, TOL
        q, k, v, pq, pk, rho = make_inputs(1, 1, N, d, 109, bq=bq, bk=bk)
    quant = case == "qat"
    dev = [to_dev(x, dt, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    out, mask, sv = sla2.forward(*dev, k_percent=kp, bq=bq, bk=bk, quant=quant, return_mask=True, saved="full")
    mask = mask[0, 0].cpu().numpy()
    ref = r.forward_saved(q[0, 0], k[0, 0], v[0, 0], bq, bk, mask, rho[0], quant=quant)
    got = {n: t[0, 0].cpu().numpy() for n, t in sv.items() if n != "qat_s_first"}
    for n in ("q_phi", "k_phi"):
        assert np.array_equal(got[n].view(np.uint32), ref[n].view(np.uint32)), n
    full = mask.all(axis=1)
    assert np.all(got["h_blocks"][full] == 0) and np.all(got["z_blocks"][full] == 0)
    for n in ("h_blocks", "z_blocks"):
        e = rel_err(got[n][~full], ref[n][~full])[0]
        assert e <= tol, (n, e)
    for n in ("o_s", "o_l"):
        assert rel_err(got[n], ref[n])[0] <= (tol if case != "f32" else 1e-4), n
    np.testing.assert_allclose(got["big_l"], ref["big_l"], atol=2e-2 if case != "f32" else 1e-4, rtol=2e-3)


@pytest.mark.skipif(oc.ref() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ["bf16", "f32"])
def test_linear_precompute_vs_reference(cuda, case):
    """sla2_linear_precompute (attention.hpp:456-475): phi(K~) bit-exact with the reference's
    k_phi; z_j per key block and the totals H = sum_j phi(K~_j)^T V_j, Z = sum_j z_j against the
    reference's phi(K~) and V (float64 sums) within the branch tolerance."""
    import torch
    r = oc.ref()
    if case == "f32":
        N, d, bq, bk, dt, tol = 1024, 64, 64, 64, torch.float32, 1e-5
        q, k, v, pq, pk, rho = make_inputs(1, 1, N, d, 110, bf16=False, bq=bq, bk=bk)
    else:
        N, d, bq, bk, dt, tol = 4096, 128, 128, 64, torch.bfloat16, TOL
        q, k, v, pq, pk, rho = make_inputs(1, 1, N, d, 111, bq=bq, bk=bk)
    res = sla2.linear_precompute(to_dev(k, dt, cuda), to_dev(v, dt, cuda), bq=bq, bk=bk)
    got = {n: t[0, 0].cpu().numpy() for n, t in res.items()}
    mask = np.ones((N // bq, N // bk), np.uint8)
    ref = r.forward_saved(q[0, 0], k[0, 0], v[0, 0], bq, bk, mask, rho[0])
    assert np.array_equal(got["k_phi"].view(np.uint32), ref["k_phi"].view(np.uint32))
    kphi = ref["k_phi"].astype(np.float64)
    zb = kphi.reshape(N // bk, bk, d).sum(axis=1)
    assert rel_err(got["z_blocks"], zb)[0] <= tol
    assert rel_err(got["z_total"], zb.sum(axis=0))[0] <= tol
    assert rel_err(got["h_total"], kphi.T @ v[0, 0].astype(np.float64))[0] <= tol
