"""Ragged N: sequence lengths that the blocks do not divide, e.g. the true
Wan2.1 shapes N = 32760 (1.3B) and N = 75600 (14B).

The reference rejects them (attention.hpp:39-41, matrix.hpp:176-179), so the semantics are an
extension, restated in the C oracle (sla2o_*_ragged, oracle/sla2_oracle_body.h):
  * tm = ceil(N / bq), tn = ceil(N / bk); the last query / key block is partial;
  * mean_pool averages a partial block over its own rows (the router's pooled Q / K~);
  * the partial key block contributes only its real keys (S, P, PV, h_j, z_j); the partial
    query block produces only its real rows.

The extension is pinned three ways (CPU): it equals the unmodified reference wherever the
reference is defined (N divisible); it equals an independent dense float64 restatement of the
definition above (numpy, below); its pooling equals numpy means. The GPU path is then checked
against it (mask bit-exact, outputs within the bf16 tolerance).
"""
import numpy as np
import pytest

import oracle_ctypes as oc

P = oc.port()
R = oc.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built (no /root/reference here)")


def _case(n, d, bq, kp_seed=0, dtype=np.float64):
    q, k, v = (P.gaussian((n, d), 900 + kp_seed + i, dtype=dtype) for i in range(3))
    pq = np.eye(d, dtype=dtype) + dtype(0.05) * P.gaussian((d, d), 910 + kp_seed, dtype=dtype)
    pk = np.eye(d, dtype=dtype) + dtype(0.05) * P.gaussian((d, d), 911 + kp_seed, dtype=dtype)
    rho = P.uniform((-(-n // bq),), 912 + kp_seed, dtype=dtype)
    return q, k, v, pq, pk, rho


@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("quant", [False, True])
def test_ragged_equals_reference_when_divisible(dtype, quant):
    n, d, bq, bk, kp = 256, 32, 32, 16, 10.0
    q, k, v, pq, pk, rho = _case(n, d, bq, dtype=dtype)
    a = P.attention_ragged(q, k, v, bq, bk, pq, pk, rho, kp, quant=quant)
    b = R.attention(q, k, v, bq, bk, pq, pk, rho, kp, quant=quant)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


def _softmax_rows(x):
    m = x.max(axis=1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=1, keepdims=True)


def _dense_ragged(q, k, v, bq, bk, mask, rho, smooth=True):
    """Independent float64 restatement of the ragged definition (dense N x N)."""
    n, d = q.shape
    kt = k - k.mean(axis=0) if smooth else k
    qb = np.arange(n) // bq
    kb = np.arange(n) // bk
    keep = mask[qb][:, kb].astype(bool)
    s = (q @ kt.T) / np.sqrt(d)
    s = np.where(keep, s, -np.inf)
    o_s = _softmax_rows(s) @ v
    lin = _softmax_rows(q) @ _softmax_rows(kt).T
    lin = np.where(keep, 0.0, lin)
    den = lin.sum(axis=1, keepdims=True)
    o_l = np.divide(lin @ v, den, out=np.zeros((n, d)), where=den != 0)
    full = mask.all(axis=1)[qb]
    a = np.clip(1.0 / (1.0 + np.exp(-rho[qb])), np.finfo(np.float64).tiny, 1 - np.finfo(np.float64).eps / 2)
    a = np.where(full, 1.0, a)[:, None]
    return a * o_s + (1 - a) * o_l


@pytest.mark.parametrize("n,bq,bk,kp", [(100, 16, 8, 30.0), (67, 8, 16, 25.0), (129, 32, 32, 50.0), (8, 16, 16, 100.0)])
def test_ragged_matches_dense_definition(n, bq, bk, kp):
    d = 8
    q, k, v, pq, pk, rho = _case(n, d, bq, kp_seed=n)
    out, mask, o_s, o_l, big_l = P.attention_ragged(q, k, v, bq, bk, pq, pk, rho, kp)
    assert mask.shape == (-(-n // bq), -(-n // bk))
    kappa = P.topk_budget(kp, mask.shape[1])
    assert (mask.sum(axis=1) == kappa).all()
    ref = _dense_ragged(q, k, v, bq, bk, mask, rho)
    assert np.abs(out - ref).max() <= 1e-10


def test_ragged_pooling_is_mean_of_real_rows():
    n, d, bq, bk = 70, 8, 16, 8
    q, k, v, pq, pk, rho = _case(n, d, bq)
    eye = np.eye(d)
    pc = np.empty((-(-n // bq), -(-n // bk)))
    assert P._block_scores_ragged_d(q, k, n, d, eye, eye, 0.1, bq, bk, pc) == 0
    qbar = np.stack([q[i:i + bq].mean(axis=0) for i in range(0, n, bq)])
    kbar = np.stack([k[j:j + bk].mean(axis=0) for j in range(0, n, bk)])
    ref = _softmax_rows(qbar @ kbar.T / np.sqrt(d))
    assert np.abs(pc - ref).max() <= 1e-12


def test_ragged_rejected_by_reference_api():
    """The reference-API oracle keeps the reference's shape_error for N % block != 0."""
    q, k, v, pq, pk, rho = _case(100, 8, 16)
    with pytest.raises(oc.ShapeError):
        P.attention(q, k, v, 16, 8, pq, pk, rho, 30.0)


# ----------------------------------------------------------------------------- GPU (bf16 path)
def _gpu_case(B, H, N, seed):
    from sla2_testlib import make_inputs
    rng = np.random.default_rng(seed)
    q, k, v, pq, pk, _ = make_inputs(B, H, -(-N // 128) * 128, 128, seed)
    q, k, v = (np.ascontiguousarray(x[:, :, :N]) for x in (q, k, v))
    rho = rng.uniform(-1, 1, (H, -(-N // 128))).astype(np.float32)
    return q, k, v, pq, pk, rho


@pytest.mark.gpu
@pytest.mark.parametrize("N,H,kp,seed", [(4000, 2, 5.0, 1), (1000, 1, 20.0, 2), (32760, 1, 3.0, 3), (75600, 1, 3.0, 4),
                                         (8200, 2, 100.0, 5)])
def test_ragged_gpu_vs_oracle(cuda, N, H, kp, seed):
    import torch
    import paper_2602_12675_b200 as sla2
    from sla2_testlib import rel_err, to_dev
    B = 1
    q, k, v, pq, pk, rho = _gpu_case(B, H, N, seed)
    out, mask, sv = sla2.forward(to_dev(q, torch.bfloat16, cuda), to_dev(k, torch.bfloat16, cuda),
                                 to_dev(v, torch.bfloat16, cuda), to_dev(pq, torch.float32, cuda),
                                 to_dev(pk, torch.float32, cuda), to_dev(rho, torch.float32, cuda), k_percent=kp,
                                 return_mask=True, saved=True)
    out, mask = out.float().cpu().numpy(), mask.cpu().numpy()
    assert mask.shape == (B, H, -(-N // 128), -(-N // 64))
    for h in range(H):
        r_out, r_mask, r_os, r_ol, r_l = P.attention_ragged(q[0, h], k[0, h], v[0, h], 128, 64, pq[h], pk[h], rho[h], kp)
        assert np.array_equal(mask[0, h], r_mask), f"ragged mask differs (head {h})"
        assert rel_err(out[0, h], r_out)[0] <= 1e-2
        assert rel_err(sv["o_s"].cpu().numpy()[0, h], r_os)[0] <= 1e-2
        if not r_mask.all():
            assert rel_err(sv["o_l"].cpu().numpy()[0, h], r_ol)[0] <= 1e-2
    assert np.isfinite(out).all()


@pytest.mark.gpu
def test_ragged_heads_do_not_bleed(cuda):
    """A ragged head's tail reads zeros, not the next head's rows: head 0 of a 2-head call equals
    the same head computed alone."""
    import torch
    import paper_2602_12675_b200 as sla2
    from sla2_testlib import to_dev
    N = 1000
    q, k, v, pq, pk, rho = _gpu_case(1, 2, N, 7)
    dev = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    both = sla2.forward(*dev, k_percent=10.0)
    one = sla2.forward(*(x[:, :1].contiguous() for x in dev[:3]), dev[3][:1].contiguous(), dev[4][:1].contiguous(),
                       dev[5][:1].contiguous(), k_percent=10.0)
    assert torch.equal(both[:, :1], one)


@pytest.mark.gpu
def test_ragged_batch_and_host_path(cuda):
    """B = 2 ragged heads: every (b, h) slice against the oracle, and the host-buffer entry point
    (pipelined per head) reproduces the device call bit for bit."""
    import torch
    import paper_2602_12675_b200 as sla2
    from sla2_testlib import rel_err, to_dev
    B, H, N, kp = 2, 2, 1000, 10.0
    q, k, v, pq, pk, rho = _gpu_case(B, H, N, 11)
    dev = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda) for x in (pq, pk, rho)]
    out, mask = sla2.forward(*dev, k_percent=kp, return_mask=True)
    for b in range(B):
        for h in range(H):
            r_out, r_mask = P.attention_ragged(q[b, h], k[b, h], v[b, h], 128, 64, pq[h], pk[h], rho[h], kp)[:2]
            assert np.array_equal(mask.cpu().numpy()[b, h], r_mask), (b, h)
            assert rel_err(out.float().cpu().numpy()[b, h], r_out)[0] <= 1e-2, (b, h)
    host = [x.cpu().pin_memory() for x in dev]
    hout, hmask = sla2.forward_host(*host, k_percent=kp, return_mask=True)
    assert torch.equal(hout, out.cpu())
    assert torch.equal(hmask, mask.cpu())
