"""The CPU oracle (oracle/sla2_oracle.c) is pinned two ways (CPU only):

1. bit-for-bit against the UNMODIFIED reference headers built into oracle/_ref
   (skipped where the reference tree was never available to build it);
2. against the reference's own known-answer tests and golden fixtures generated from the
   reference (tests/golden, made by tests/golden/make_golden.py), which need no reference tree.
"""
import os

import numpy as np
import pytest

import oracle_ctypes as oc

P = oc.port()
R = oc.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built (no /root/reference here)")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ------------------------------------------------------------------- reference KATs (no _ref needed)
def test_topk_budget_kat():
    # router.hpp:36-40; paper budgets at the Wan shapes
    assert P.topk_budget(3.0, 512) == 15
    assert P.topk_budget(3.0, 1182) == 35
    assert P.topk_budget(10.0, 64) == 6
    assert P.topk_budget(25.0, 4) == 1
    assert P.topk_budget(0.001, 100) == 1
    assert P.topk_budget(100.0, 7) == 7


def test_hard_topk_unique_max():  # test_router.cpp:58-66
    mask, kappa = P.hard_topk(np.array([[0.1, 0.5, 0.2, 0.2]]), 25.0)
    assert kappa == 1 and mask.tolist() == [[0, 1, 0, 0]]


def test_hard_topk_tie_breaks_to_lowest_column():  # test_router.cpp:68-73
    mask, _ = P.hard_topk(np.array([[0.3, 0.3, 0.2, 0.2]]), 25.0)
    assert mask.tolist() == [[1, 0, 0, 0]]


def test_hard_topk_matches_full_sort_oracle():  # test_router.cpp:75-89
    pc = P.uniform((8, 16), 111)
    mask, _ = P.hard_topk(pc, 25.0)
    for i in range(8):
        order = sorted(range(16), key=lambda j: (-pc[i, j], j))
        exp = np.zeros(16, np.uint8)
        exp[order[:4]] = 1
        assert np.array_equal(mask[i], exp)


def test_hard_topk_invariant_under_monotone_transforms():  # test_router.cpp:91-104
    pc = P.uniform((6, 12), 112)
    base, _ = P.hard_topk(pc, 30.0)
    e = np.exp(pc - pc.max(axis=1, keepdims=True))
    for variant in (e / e.sum(axis=1, keepdims=True), 2.0 * pc + 1.0, 37.5 * pc):
        assert np.array_equal(P.hard_topk(np.ascontiguousarray(variant), 30.0)[0], base)


def test_hard_topk_sparsity_exact_and_range():  # test_router.cpp:106-116
    mask, _ = P.hard_topk(P.uniform((5, 20), 113), 10.0)
    assert mask.sum() == 5 * 2
    with pytest.raises(oc.ShapeError):
        P.hard_topk(np.zeros((1, 4)), 0.0)
    with pytest.raises(oc.ShapeError):
        P.hard_topk(np.zeros((1, 4)), 101.0)


def test_block_scores_zero_inputs_uniform():  # test_router.cpp:12-19
    z = np.zeros((16, 4))
    pc = P.block_scores(z, z, np.eye(4), np.eye(4), 4, 2)
    assert np.all(pc == 1.0 / 8)


def test_block_scores_averaged_token_oracle():  # test_router.cpp:32-56
    n, d, bq, bk = 32, 8, 4, 2
    q, k = P.gaussian((n, d), 103), P.gaussian((n, d), 104)
    pq, pk = P.gaussian((d, d), 105), P.gaussian((d, d), 106)
    pc = P.block_scores(q, k, pq, pk, bq, bk)
    ts = (q @ pq) @ (k @ pk).T / np.sqrt(d)
    avg = ts.reshape(n // bq, bq, n // bk, bk).mean(axis=(1, 3))
    e = np.exp(avg - avg.max(axis=1, keepdims=True))
    assert np.abs(pc - e / e.sum(axis=1, keepdims=True)).max() <= 1e-10


def test_quantize_direct_formula_kat():  # test_quant.cpp:10-22
    codes, scale = P.quantize(np.array([1.0, -0.5, 0.25, 0.0]))
    assert scale == 1.0 / 127.0
    assert codes.tolist() == [127, -64, 32, 0]  # -63.5 rounds away from zero


def test_quantize_zero_block_and_scale_invariance():  # test_quant.cpp:24-37
    codes, scale = P.quantize(np.zeros(9))
    assert not codes.any() and scale > 0
    x = P.gaussian((6, 6), 201)
    assert np.array_equal(P.quantize(x)[0], P.quantize(10.0 * x)[0])


def test_quantize_round_trip_within_half_scale():  # test_quant.cpp:39-48
    for seed in (202, 203, 204):
        x = P.gaussian((8, 8), seed, 3.0)
        codes, scale = P.quantize(x)
        assert np.abs(codes * scale - x).max() <= scale / 2 + 1e-15


def test_smooth_k_properties():  # test_quant.cpp:87-112
    k = np.full((6, 3), 2.5)
    kt, mu = P.smooth_k(k)
    assert np.all(kt == 0) and np.all(mu == 2.5)
    k = P.gaussian((10, 4), 209)
    k0 = k - k.mean(axis=0)
    assert np.abs(P.smooth_k(k0)[0] - k0).max() <= 1e-15


def _small_case(seed, n=64, d=8, bq=8, bk=4, k_percent=25.0, dtype=np.float64):
    q, k, v = (P.gaussian((n, d), seed + i, dtype=dtype) for i in range(3))
    kt = P.smooth_k(k)[0]
    mask, _ = P.hard_topk(P.block_scores(q, kt, np.eye(d, dtype=dtype), np.eye(d, dtype=dtype), bq, bk), k_percent)
    return q, k, v, mask


@pytest.mark.parametrize("seed", [351, 352, 353])
@pytest.mark.parametrize("k_percent", [10.0, 25.0, 50.0])
def test_blockwise_matches_naive(seed, k_percent):  # test_attention.cpp:215-230
    q, k, v, mask = _small_case(seed, k_percent=k_percent)
    rho = np.zeros(64 // 8)
    naive = P.forward_naive(q, k, v, 8, 4, mask, rho)[0]
    blockwise = P.forward_blockwise(q, k, v, 8, 4, mask, rho)[0]
    assert np.abs(naive - blockwise).max() <= 1e-10


def test_blockwise_single_precision_matches_naive():  # test_attention.cpp:232-241
    q, k, v, mask = _small_case(354, dtype=np.float32)
    rho = np.zeros(8, np.float32)
    assert np.abs(P.forward_naive(q, k, v, 8, 4, mask, rho)[0] - P.forward_blockwise(q, k, v, 8, 4, mask, rho)[0]).max() <= 1e-4


def test_full_mask_high_alpha_is_full_attention():  # test_attention.cpp:167-174
    n, d = 32, 8
    q, k, v = (P.gaussian((n, d), 341 + i) for i in range(3))
    mask = np.ones((n // 4, n // 4), np.uint8)
    out = P.forward_naive(q, k, v, 4, 4, mask, np.full(8, 40.0))[0]
    s = q @ k.T / np.sqrt(d)
    p = np.exp(s - s.max(axis=1, keepdims=True))
    ref = (p / p.sum(axis=1, keepdims=True)) @ v
    assert np.abs(out - ref).max() <= 1e-6


def test_empty_complement_forces_sparse_branch():  # test_attention.cpp:176-184
    n, d = 32, 8
    q, k, v = (P.gaussian((n, d), 342 + i) for i in range(3))
    mask = np.ones((8, 8), np.uint8)
    out, o_s, o_l, _ = P.forward_blockwise(q, k, v, 4, 4, mask, np.full(8, -5.0))
    assert np.array_equal(out, o_s)


def test_smoothing_leaves_sparse_branch_unchanged():  # test_attention.cpp:270-279
    n, d = 32, 8
    q, k, v = (P.gaussian((n, d), 357 + i) for i in range(3))
    mask, _ = P.hard_topk(P.uniform((8, 8), 358), 3 / 8 * 100)
    rho = np.zeros(8)
    _, os1, ol1, _ = P.forward_blockwise(q, k, v, 4, 4, mask, rho, smooth=True)
    _, os2, ol2, _ = P.forward_blockwise(q, k, v, 4, 4, mask, rho, smooth=False)
    assert np.abs(os1 - os2).max() <= 1e-10
    assert np.abs(ol1 - ol2).max() > 1e-10


def test_empty_mask_row_raises():  # test_attention.cpp:305-311
    n, d = 16, 4
    q, k, v = (P.gaussian((n, d), 362 + i) for i in range(3))
    mask = np.zeros((4, 4), np.uint8)
    mask[0, 0] = mask[1, 1] = mask[2, 2] = 1
    with pytest.raises(oc.ShapeError):
        P.forward_blockwise(q, k, v, 4, 4, mask, np.zeros(4))


def test_qat_deviation_band():  # test_attention.cpp:313-323
    n, d = 32, 8
    q, k, v = (P.gaussian((n, d), 363 + i) for i in range(3))
    mask, _ = P.hard_topk(P.uniform((8, 8), 364), 2 / 8 * 100)
    rho = np.zeros(8)
    exact = P.forward_blockwise(q, k, v, 4, 4, mask, rho)[0]
    quant = P.forward_blockwise(q, k, v, 4, 4, mask, rho, quant=True)[0]
    dev = np.abs(exact - quant).max()
    assert 0 < dev <= 5e-2


# ------------------------------------------------------------------- bit-exact vs the reference itself
@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rng_streams_match_libstdcxx(dtype):
    for seed in (0, 7, 351):
        assert np.array_equal(P.gaussian((999,), seed, 1.7, dtype), R.gaussian((999,), seed, 1.7, dtype))
        assert np.array_equal(P.uniform((999,), seed, -2, 3, dtype), R.uniform((999,), seed, -2, 3, dtype))


@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("quant", [False, True])
@pytest.mark.parametrize("n,d,bq,bk,kp", [(256, 32, 32, 16, 10.0), (512, 64, 64, 32, 3.0), (64, 8, 8, 4, 50.0)])
def test_port_bitexact_vs_reference(dtype, quant, n, d, bq, bk, kp):
    q, k, v = (P.gaussian((n, d), 10 + i, dtype=dtype) for i in range(3))
    pq = np.eye(d, dtype=dtype) + dtype(0.05) * P.gaussian((d, d), 20, dtype=dtype)
    pk = np.eye(d, dtype=dtype) + dtype(0.05) * P.gaussian((d, d), 21, dtype=dtype)
    rho = P.uniform((n // bq,), 22, dtype=dtype)
    a = P.attention(q, k, v, bq, bk, pq, pk, rho, kp, quant=quant)
    b = R.attention(q, k, v, bq, bk, pq, pk, rho, kp, quant=quant)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


@needs_ref
def test_port_bitexact_vs_reference_bf16_inputs_wan_block_shape():
    """bq = 128, bk = 64, d = 128 on bf16-valued float inputs (the GPU configuration)."""
    from sla2_testlib import make_inputs
    q, k, v, pq, pk, rho = make_inputs(1, 1, 2048, 128, seed=3)
    a = P.attention(q[0, 0], k[0, 0], v[0, 0], 128, 64, pq[0], pk[0], rho[0], 5.0)
    b = R.attention(q[0, 0], k[0, 0], v[0, 0], 128, 64, pq[0], pk[0], rho[0], 5.0)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8))


# ------------------------------------------------------------------- golden fixtures from the reference
def _golden_files():
    if not os.path.isdir(GOLDEN):
        return []
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz") and not f.startswith(("backward_", "soft_")))


@pytest.mark.parametrize("name", _golden_files())
def test_port_matches_reference_golden(name):
    g = np.load(os.path.join(GOLDEN, name))
    dt = g["q"].dtype
    out, mask, o_s, o_l, big_l = P.attention(g["q"], g["k"], g["v"], int(g["bq"]), int(g["bk"]), g["proj_q"],
                                             g["proj_k"], g["rho"], float(g["k_percent"]), quant=bool(g["quant"]))
    assert np.array_equal(mask, g["mask"])
    for a, b in ((out, g["out"]), (o_s, g["o_s"]), (o_l, g["o_l"]), (big_l, g["big_l"])):
        assert a.dtype == dt and np.array_equal(a.view(np.uint8), b.view(np.uint8))
