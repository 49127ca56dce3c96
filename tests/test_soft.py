"""Stage-1 soft routing: the device soft_topk (router.hpp:126-190) and the
SoftMask forward (attention.hpp:484-558) against the UNMODIFIED reference (oracle/_ref, which
travels to the GPU box prebuilt) and against fixtures it wrote (tests/golden/soft_*.npz).

Tolerances: soft_topk values |gpu - ref| <= 1e-6 (both bisect in double; the row sum's order
differs, which moves lambda by < 1e-6 / (sum sigma')); the forward's outputs 2e-5 normwise
(max|gpu - ref| <= 2e-5 max|ref|) -- fp32 with a different accumulation order than the
reference's serial loops. The reference's own soft_topk tests (test_router.cpp:118-165) are
restated on the device path as property tests."""
import os

import numpy as np
import pytest

import oracle_ctypes as oc
import paper_2602_12675_b200 as sla2

R = oc.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built (no /root/reference here)")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL_V = 1e-6
TOL = 2e-5


def _rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def _soft_goldens():
    return sorted(os.path.join(GOLDEN, f) for f in os.listdir(GOLDEN) if f.startswith("soft_") and f.endswith(".npz"))


def _naive_soft(q, k, v, bq, bk, w, rho, smooth=True):
    """Dense restatement of the SoftMask forward in float64: the sparse branch is a softmax whose
    key-block j terms are weighted by w_ij, the linear branch weights phi(K~_j) by 1 - w_ij."""
    q, k, v = (np.asarray(x, np.float64) for x in (q, k, v))
    n, d = q.shape
    kt = k - k.mean(axis=0) if smooth else k
    wb = np.repeat(np.repeat(np.asarray(w, np.float64), bq, axis=0), bk, axis=1)
    s = q @ kt.T / np.sqrt(d)
    e = np.exp(s - s.max(axis=1, keepdims=True)) * wb
    o_s = e @ v / e.sum(axis=1, keepdims=True)
    sm = lambda x: np.exp(x - x.max(axis=1, keepdims=True)) / np.exp(x - x.max(axis=1, keepdims=True)).sum(1, keepdims=True)  # noqa: E731
    pq, pk = sm(q), sm(kt)
    a = (pq @ pk.T) * (1.0 - wb)
    o_l = a @ v / a.sum(axis=1, keepdims=True)
    alpha = np.repeat(1.0 / (1.0 + np.exp(-np.asarray(rho, np.float64))), bq)[:, None]
    return alpha * o_s + (1 - alpha) * o_l, o_s, o_l


# ---------------------------------------------------------------- CPU: the reference binding
@needs_ref
def test_reference_soft_binding_cpu():
    """The shim's soft_topk meets the budget and its SoftMask forward equals the dense
    restatement (the reference's SoftRoutingMatchesNaive, test_attention.cpp:282-292)."""
    P = oc.port()
    n, d, bq, bk = 32, 8, 4, 4
    q, k, v = (P.gaussian((n, d), 359 + i) for i in range(3))
    kt, _ = R.smooth_k(k)
    pc = R.block_scores(q, kt, np.eye(d), np.eye(d), bq, bk)
    values, lambdas = R.soft_topk(pc, 25.0, 0.1)
    assert np.abs(values.sum(axis=1) - 2.0).max() <= 1e-6
    rho = np.full(n // bq, np.log(0.3 / 0.7))
    out, o_s, o_l, _ = R.forward_soft(q, k, v, bq, bk, values, rho)
    ref, rs, rl = _naive_soft(q, k, v, bq, bk, values, rho)
    assert np.abs(o_s - rs).max() <= 1e-10
    assert np.abs(o_l - rl).max() <= 1e-10
    assert np.abs(out - ref).max() <= 1e-10


@needs_ref
@pytest.mark.parametrize("path", _soft_goldens(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_soft_goldens_reproduce_cpu(path):
    """The committed fixtures are what the reference computes today."""
    z = np.load(path)
    bq, bk = int(z["bq"]), int(z["bk"])
    values, lambdas = R.soft_topk(z["pc"], float(z["k_percent"]), float(z["tau"]))
    assert np.array_equal(values, z["values"]) and np.array_equal(lambdas, z["lambdas"])
    out = R.forward_soft(z["q"], z["k"], z["v"], bq, bk, values, z["rho"])[0]
    assert np.array_equal(out, z["out"])


# ---------------------------------------------------------------- GPU: soft_topk
def _t(x, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("tm,tn,kp,tau,seed", [(64, 32, 25.0, 0.1, 1), (16, 512, 3.0, 0.05, 2),
                                               (8, 2048, 3.0, 0.1, 3), (37, 100, 50.0, 1e-3, 4)])
def test_soft_topk_vs_reference(cuda, tm, tn, kp, tau, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2, 3, tm, tn))
    pc = (np.exp(x) / np.exp(x).sum(-1, keepdims=True)).astype(np.float32)  # row-softmaxed scores
    values, lambdas = sla2.soft_topk(_t(pc, cuda), k_percent=kp, tau=tau)
    values, lambdas = values.cpu().numpy(), lambdas.cpu().numpy()
    kappa = R.topk_budget(kp, tn)
    for b in range(2):
        for h in range(3):
            rv, rl = R.soft_topk(pc[b, h], kp, tau)
            assert np.abs(values[b, h] - rv).max() <= TOL_V
            assert np.abs(lambdas[b, h] - rl).max() <= 1e-5 * max(1.0, np.abs(rl).max())
            assert np.abs(values[b, h].astype(np.float64).sum(-1) - kappa).max() <= 1e-6 * tn + 1e-6


@pytest.mark.gpu
def test_soft_topk_reference_properties(cuda):
    """test_router.cpp:118-165 on the device: uniform row -> kappa/tn; small tau -> the hard
    indicator; values inside [0, 1]; monotone within a row."""
    v, _ = sla2.soft_topk(_t(np.full((1, 1, 1, 4), 0.7), cuda), k_percent=50.0, tau=0.1)
    assert np.abs(v.cpu().numpy() - 0.5).max() <= 1e-6
    rng = np.random.default_rng(121)
    grid = np.stack([rng.permutation(8) + 1.0 for _ in range(4)]) / 8.0
    v, _ = sla2.soft_topk(_t(grid[None, None], cuda), k_percent=25.0, tau=1e-3)
    hard = (grid >= np.sort(grid, axis=1)[:, -2:-1]).astype(np.float64)  # kappa = 2, distinct entries
    assert np.abs(v.cpu().numpy()[0, 0] - hard).max() <= 1e-3
    x = rng.uniform(-1, 1, (8, 16))
    pc = np.exp(x) / np.exp(x).sum(1, keepdims=True)
    v = sla2.soft_topk(_t(pc[None, None], cuda), k_percent=20.0, tau=1e-3)[0].cpu().numpy()[0, 0]
    # strictly inside (0, 1) in double; the fp32 cast (the reference's T = float) rounds the clamp
    # bounds DBL_MIN and 1 - eps/2 to 0 and 1
    assert (v >= 0).all() and (v <= 1).all() and np.isfinite(v).all()
    v = sla2.soft_topk(_t(pc[None, None], cuda), k_percent=30.0, tau=0.1)[0].cpu().numpy()[0, 0]
    pcf = pc.astype(np.float32)
    for i in range(8):
        order = np.argsort(pcf[i], kind="stable")
        assert np.all(np.diff(v[i][order]) >= 0)


@pytest.mark.gpu
def test_soft_topk_errors(cuda):
    """Non-convergence raises numeric_error like the reference (router.hpp:181-184): three tied
    maxima at tau = 1e-15 cannot share a budget of 2 within 1e-6 in double."""
    pc = _t(np.array([1, 1, 1, 0.0])[None, None, None], cuda)
    with pytest.raises(sla2.NumericError):
        sla2.soft_topk(pc, k_percent=50.0, tau=1e-15)
    with pytest.raises(sla2.NumericError):  # tau must be positive (router.hpp:131)
        sla2.soft_topk(pc, k_percent=50.0, tau=0.0)
    # no k_percent range check: topk_budget clamps to kappa = 1 (router.hpp:36-40, 130-133)
    v, _ = sla2.soft_topk(pc, k_percent=0.0, tau=0.1)
    assert abs(float(v.sum()) - 1.0) < 1e-5


@needs_ref
def test_soft_topk_nonconvergence_matches_reference_cpu():
    with pytest.raises(oc.OracleError):
        R.soft_topk(np.array([[1, 1, 1, 0.0]], np.float32), 50.0, 1e-15)


# ---------------------------------------------------------------- GPU: the SoftMask forward
@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("N,H,d,bq,bk,kp,tau,smooth,seed", [(1024, 2, 64, 64, 64, 25.0, 0.1, True, 1),
                                                             (512, 1, 64, 32, 64, 10.0, 0.05, True, 2),
                                                             (512, 1, 32, 64, 32, 30.0, 0.1, False, 3),
                                                             (256, 2, 16, 16, 16, 3.0, 1e-3, True, 4)])
def test_forward_soft_vs_reference(cuda, N, H, d, bq, bk, kp, tau, smooth, seed):
    """The whole stage-1 chain on the device (router pc -> soft_topk -> SoftMask forward)
    against the reference's chain on the same inputs (stage1_record_grads, training.hpp:186-201)."""
    import torch
    from sla2_testlib import make_inputs, to_dev
    q, k, v, pq, pk, rho = make_inputs(1, H, N, d, seed, bf16=False, bq=bq, bk=bk)
    dev = [to_dev(x, torch.float32, cuda) for x in (q, k, v, pq, pk, rho)]
    pc = sla2.router(dev[0], dev[1], dev[3], dev[4], k_percent=kp, bq=bq, bk=bk, smooth=smooth)[0]
    values, _ = sla2.soft_topk(pc, k_percent=kp, tau=tau)
    out, sv = sla2.forward_soft(dev[0], dev[1], dev[2], dev[5], values, bq=bq, bk=bk, smooth=smooth, saved=True)
    for h in range(H):
        kt = R.smooth_k(k[0, h])[0] if smooth else k[0, h]
        rpc = R.block_scores(q[0, h], kt, pq[h], pk[h], bq, bk)
        assert np.array_equal(pc.cpu().numpy()[0, h], rpc)  # the router is bit-exact
        rv, _ = R.soft_topk(rpc, kp, tau)
        assert np.abs(values.cpu().numpy()[0, h] - rv).max() <= TOL_V
        ro, ros, rol, rl = R.forward_soft(q[0, h], k[0, h], v[0, h], bq, bk, rv, rho[h], smooth=smooth)
        assert _rel(out.cpu().numpy()[0, h], ro) <= TOL, h
        assert _rel(sv["o_s"].cpu().numpy()[0, h], ros) <= TOL, h
        assert _rel(sv["o_l"].cpu().numpy()[0, h], rol) <= TOL, h
        assert np.abs(sv["big_l"].cpu().numpy()[0, h] - rl).max() <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("path", _soft_goldens(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_forward_soft_vs_reference_golden(cuda, path):
    """Against the fixtures the reference wrote: no oracle/_ref needed."""
    import torch
    z = np.load(path)
    bq, bk, kp, tau = int(z["bq"]), int(z["bk"]), float(z["k_percent"]), float(z["tau"])
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x))[None, None].to(cuda)  # noqa: E731
    q, k, v = t(z["q"]), t(z["k"]), t(z["v"])
    pq, pk = (torch.from_numpy(z[n])[None].to(cuda) for n in ("proj_q", "proj_k"))
    rho = torch.from_numpy(z["rho"])[None].to(cuda)
    pc = sla2.router(q, k, pq, pk, k_percent=kp, bq=bq, bk=bk)[0]
    assert np.array_equal(pc.cpu().numpy()[0, 0], z["pc"])
    values, lambdas = sla2.soft_topk(pc, k_percent=kp, tau=tau)
    assert np.abs(values.cpu().numpy()[0, 0] - z["values"]).max() <= TOL_V
    out, sv = sla2.forward_soft(q, k, v, rho, values, bq=bq, bk=bk, saved=True)
    assert _rel(out.cpu().numpy()[0, 0], z["out"]) <= TOL
    assert _rel(sv["o_s"].cpu().numpy()[0, 0], z["o_s"]) <= TOL
    assert _rel(sv["o_l"].cpu().numpy()[0, 0], z["o_l"]) <= TOL


@pytest.mark.gpu
def test_forward_soft_hard_values_equal_hard_forward(cuda):
    """A 0/1 SoftMask reproduces the hard-mask fp32 forward where no row is full (both
    branches are then the same sums; attention.hpp:490-491)."""
    import torch
    from sla2_testlib import make_inputs, to_dev
    q, k, v, pq, pk, rho = make_inputs(1, 2, 512, 64, 9, bf16=False, bq=64, bk=64)
    dev = [to_dev(x, torch.float32, cuda) for x in (q, k, v, pq, pk, rho)]
    out, mask = sla2.forward(*dev, k_percent=25.0, bq=64, bk=64, return_mask=True)
    soft = sla2.forward_soft(dev[0], dev[1], dev[2], dev[5], mask.float(), bq=64, bk=64)
    assert _rel(soft.cpu().numpy(), out.cpu().numpy()) <= TOL


@pytest.mark.gpu
def test_forward_soft_contract(cuda):
    import torch
    x = torch.zeros((1, 1, 256, 128), device=cuda)
    with pytest.raises(sla2.ContractError):  # d = 128 > 64 on this path
        sla2.forward_soft(x, x, x, torch.zeros((1, 4), device=cuda), torch.zeros((1, 1, 4, 4), device=cuda))
    y = torch.zeros((1, 1, 256, 64), device=cuda)
    with pytest.raises(sla2.ShapeError):
        sla2.forward_soft(y, y, y, torch.zeros((1, 4), device=cuda), torch.zeros((1, 1, 4, 3), device=cuda))
    with pytest.raises(sla2.ShapeError):  # N not divisible
        z = torch.zeros((1, 1, 250, 64), device=cuda)
        sla2.forward_soft(z, z, z, torch.zeros((1, 4), device=cuda), torch.zeros((1, 1, 4, 4), device=cuda))


# ---------------------------------------------------------------- soft_topk_backward
@needs_ref
def test_soft_topk_backward_reference_properties_cpu():
    """test_router.cpp:173-205 through the shim: zero upstream gives zero; doubling tau halves it."""
    rng = np.random.default_rng(131)
    pc = rng.uniform(-1, 1, (3, 6)).astype(np.float32)
    assert np.all(R.soft_topk_backward(pc, 50.0, 0.2, np.zeros((3, 6), np.float32)) == 0)
    up = rng.uniform(-1, 1, (3, 6)).astype(np.float32)
    g1 = R.soft_topk_backward(pc.astype(np.float64), 50.0, 0.2, up.astype(np.float64))
    v, _ = R.soft_topk(pc.astype(np.float64), 50.0, 0.2)
    assert np.abs(g1 - up * v * (1 - v) / 0.2).max() <= 1e-15


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("tm,tn,kp,tau,seed", [(64, 32, 25.0, 0.1, 1), (16, 512, 3.0, 0.05, 2)])
def test_soft_topk_backward_vs_reference(cuda, tm, tn, kp, tau, seed):
    """Bit-exact against the reference's soft_topk_backward given the same values (same
    elementwise order, no FMA)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((2, 2, tm, tn))
    pc = (np.exp(x) / np.exp(x).sum(-1, keepdims=True)).astype(np.float32)
    up = rng.standard_normal((2, 2, tm, tn)).astype(np.float32)
    values, _ = sla2.soft_topk(_t(pc, cuda), k_percent=kp, tau=tau)
    g = sla2.soft_topk_backward(values, _t(up, cuda), tau=tau).cpu().numpy()
    vals = values.cpu().numpy()
    for b in range(2):
        for h in range(2):
            rv, _ = R.soft_topk(pc[b, h], kp, tau)
            rg = R.soft_topk_backward(pc[b, h], kp, tau, up[b, h])
            if np.array_equal(vals[b, h], rv):  # same values -> same gradient bits
                assert np.array_equal(g[b, h], rg), (b, h)
            else:
                assert np.abs(g[b, h] - rg).max() <= 1e-5 * max(1.0, np.abs(rg).max())


@pytest.mark.gpu
@needs_ref
def test_forward_soft_batch_heads_layout(cuda):
    """B = 2, H = 3 (per-head rho rows, (b, h) slices) with and without smoothing: every slice
    against the reference's SoftMask forward on the same values."""
    import torch
    from sla2_testlib import make_inputs, to_dev
    B, H, N, d, bq, bk = 2, 3, 256, 32, 32, 32
    for smooth in (True, False):
        q, k, v, pq, pk, rho = make_inputs(B, H, N, d, 21, bf16=False, bq=bq, bk=bk)
        rng = np.random.default_rng(22)
        x = rng.standard_normal((B, H, N // bq, N // bk))
        pc = (np.exp(x) / np.exp(x).sum(-1, keepdims=True)).astype(np.float32)
        values, _ = sla2.soft_topk(_t(pc, cuda), k_percent=25.0, tau=0.1)
        dev = [to_dev(t, torch.float32, cuda) for t in (q, k, v, rho)]
        out = sla2.forward_soft(dev[0], dev[1], dev[2], dev[3], values, bq=bq, bk=bk, smooth=smooth).cpu().numpy()
        vals = values.cpu().numpy()
        for b in range(B):
            for h in range(H):
                ro = R.forward_soft(q[b, h], k[b, h], v[b, h], bq, bk, vals[b, h], rho[h], smooth=smooth)[0]
                assert _rel(out[b, h], ro) <= TOL, (smooth, b, h)
