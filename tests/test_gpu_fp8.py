"""The FP8 P/V low-bit mode (quant="fp8", SLA2_QUANT_FP8PV): BASELINE configs[2]'s "FP8 PV" on
kind::f8f6f4 -- E4M3 P (unscaled: P <= 2^8 under the lazy rescale), E4M3 V with one scale per
head, E4M3 448 phi(K~) -- with bf16 Q K^T and fp32 accumulation in TMEM.

The reference is INT8-only (quant.hpp:15-19), so this mode has no bit-level oracle: the router
(mask, kept-block lists) is the same exact code as every other mode and must stay bit-exact,
and `out` is checked against the unquantized reference forward (attention.hpp:423-560).

Tolerance: E4M3 keeps 3 mantissa bits (relative rounding error up to 2^-4), and O = sum_j P_j V_j
over random V is a cancelling sum as large as its own rounding noise, so the relative error of
O does not shrink with the number of keys: measured 3.0-3.6e-2 normwise L2 (3.6-6.6e-2 max) on
B200, against 2-3e-3 for the bf16 path. The bar here is therefore FP8_L2 = 5e-2 (L2 normwise)
and FP8_MAX = 1e-1 (max normwise), wider than the 1e-2 bf16 / INT8-QAT bar; the test also
prints the reference's own INT8 QAT deviation from the unquantized forward for comparison."""
import numpy as np
import pytest

import paper_2602_12675_b200 as sla2
from sla2_testlib import mask_to_idx, rel_err, to_dev

TOL = 1e-2
FP8_L2 = 5e-2
FP8_MAX = 1e-1


def _inputs(H, N, seed, vscale=1.0):
    rng = np.random.default_rng(seed)
    npad = -(-N // 128) * 128
    from sla2_testlib import make_inputs
    q, k, v, pq, pk, _ = make_inputs(1, H, npad, 128, seed)
    q, k, v = (np.ascontiguousarray(x[:, :, :N]) for x in (q, k, v))
    v = (v * vscale).astype(np.float32)
    rho = rng.uniform(-1, 1, (H, -(-N // 128))).astype(np.float32)
    return q, k, v, pq, pk, rho


def _run(cuda, q, k, v, pq, pk, rho, kp, quant):
    import torch
    args = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda)
                                                                    for x in (pq, pk, rho)]
    out, mask, idx = sla2.forward(*args, k_percent=kp, quant=quant, return_mask=True, return_idx=True)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), mask.cpu().numpy(), idx.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("N,H,kp,seed,vscale", [(4096, 2, 3.0, 301, 1.0), (8192, 2, 10.0, 302, 1.0),
                                                (2048, 1, 50.0, 303, 1.0), (8200, 2, 3.0, 304, 1.0),
                                                (4096, 1, 3.0, 305, 37.0), (4096, 1, 3.0, 306, 1e-3),
                                                # odd kappa (a single-block last pair: 3 of 64 blocks,
                                                # 9 of 128) and kappa = tn (no linear branch)
                                                (4096, 1, 5.0, 307, 1.0), (8192, 1, 7.0, 308, 1.0),
                                                (4096, 1, 100.0, 309, 1.0)])
def test_fp8pv_vs_reference(cuda, N, H, kp, seed, vscale):
    """Masks bit-exact (same router as the bf16 path) and out within the FP8 bar of the
    reference's unquantized forward, including ragged N and V far from unit scale."""
    from sla2_testlib import oracle_attention_any, oracle_router_any
    q, k, v, pq, pk, rho = _inputs(H, N, seed, vscale)
    out, mask, idx = _run(cuda, q, k, v, pq, pk, rho, kp, "fp8")
    out16, mask16, _ = _run(cuda, q, k, v, pq, pk, rho, kp, False)
    assert np.array_equal(mask, mask16)
    for h in range(H):
        _, rmask, _, _ = oracle_router_any(q[0, h], k[0, h], pq[h], pk[h], 128, 64, kp)
        assert np.array_equal(mask[0, h], rmask), h
        assert np.array_equal(idx[0, h], np.stack(mask_to_idx(rmask))), h
        r_out = oracle_attention_any(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], 128, 64, kp)[0]
        e8, e16 = rel_err(out[0, h], r_out), rel_err(out16[0, h], r_out)
        e_i8 = (rel_err(oracle_attention_any(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], 128, 64, kp,
                                             quant=True)[0], r_out) if N % 128 == 0 else (float("nan"),) * 2)
        print(f"N={N} h={h} fp8 max/l2 {e8[0]:.2e}/{e8[1]:.2e}  bf16 {e16[0]:.2e}/{e16[1]:.2e}  "
              f"reference INT8 QAT {e_i8[0]:.2e}/{e_i8[1]:.2e}")
        assert e16[0] <= TOL, (h, e16)
        assert e8[1] <= FP8_L2 and e8[0] <= FP8_MAX, (h, e8, e16)


@pytest.mark.gpu
def test_fp8pv_cfg3_full_call(cuda):
    """The benchmarked call (bench.py cfg3fp8): B=1, H=12, N=32760; every mask vs the oracle
    router, two output heads vs the oracle forward."""
    from sla2_testlib import oracle_attention_any, oracle_router_any
    H, N, kp = 12, 32760, 3.0
    q, k, v, pq, pk, rho = _inputs(H, N, 310)
    out, mask, idx = _run(cuda, q, k, v, pq, pk, rho, kp, "fp8")
    assert np.isfinite(out).all()
    for h in range(H):
        _, rmask, _, _ = oracle_router_any(q[0, h], k[0, h], pq[h], pk[h], 128, 64, kp)
        assert np.array_equal(mask[0, h], rmask), h
    for h in (0, H - 1):
        r_out = oracle_attention_any(q[0, h], k[0, h], v[0, h], pq[h], pk[h], rho[h], 128, 64, kp)[0]
        e8 = rel_err(out[0, h], r_out)
        assert e8[1] <= FP8_L2 and e8[0] <= FP8_MAX, (h, e8)


@pytest.mark.gpu
def test_fp8pv_rejects_saved_state(cuda):
    import torch
    q, k, v, pq, pk, rho = _inputs(1, 2048, 320)
    args = [to_dev(x, torch.bfloat16, cuda) for x in (q, k, v)] + [to_dev(x, torch.float32, cuda)
                                                                    for x in (pq, pk, rho)]
    with pytest.raises(sla2.ContractError):
        sla2.forward(*args, quant="fp8", saved=True)


def test_fp8pv_params_host():
    """Host-side validation only (no GPU): fp8 is a bf16-path mode; unknown modes are refused."""
    import ctypes as C
    p = sla2.FwdParams(1, 2, 4096, 128, 128, 64, 3.0, True, "fp8")
    assert p.c().quant == 2
    assert sla2.lib().sla2_check_params(C.byref(p.c())) == 0
    p32 = sla2.FwdParams(1, 2, 4096, 128, 128, 64, 3.0, False, "fp8")
    assert sla2.lib().sla2_check_params(C.byref(p32.c())) != 0
    ragged = sla2.FwdParams(1, 2, 8200, 128, 128, 64, 3.0, True, "fp8")
    assert sla2.lib().sla2_check_params(C.byref(ragged.c())) == 0
    with pytest.raises(sla2.ContractError):
        sla2.FwdParams(1, 2, 4096, 128, 128, 64, 3.0, True, "fp4").c()
