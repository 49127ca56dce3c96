"""C ABI checks that need no GPU: the library loads, exports every symbol include/sla2_capi.h
declares, validates parameters with the reference's error classes, and refuses to compute
without an sm_100a device (there is no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

import paper_2602_12675_b200 as sla2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sla2_capi.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sla2_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = sla2.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_version_and_budget():
    assert b"sm_100a" in sla2.lib().sla2_version()
    assert sla2.topk_budget(3.0, 512) == 15
    assert sla2.topk_budget(3.0, 1182) == 35
    assert sla2.topk_budget(0.01, 64) == 1
    assert sla2.topk_budget(100.0, 64) == 64


def test_default_params_are_the_papers():
    p = sla2._Params()
    sla2.lib().sla2_default_params(C.byref(p), 1, 12, 32768, 128)
    assert (p.bq, p.bk, p.k_percent, p.dtype, p.smooth, p.exact_mu) == (128, 64, 3.0, 1, 1, 1)
    assert abs(p.tau - 0.1) < 1e-7


@pytest.mark.parametrize("kw,err", [
    (dict(N=1000, quant=True), sla2.ShapeError),          # attention.hpp:39-41 (QAT keeps the rule)
    (dict(N=1000, bf16=False, d=64, bq=64, bk=64), sla2.ShapeError),  # and so does the fp32 path
    (dict(k_percent=0.0), sla2.ShapeError),               # router.hpp:108-110
    (dict(k_percent=101.0), sla2.ShapeError),
    (dict(tau=0.0), sla2.NumericError),                   # router.hpp:32
    (dict(d=64), sla2.ContractError),                     # bf16 kernels are d = 128 only
    (dict(bf16=False, bq=96, N=3072), sla2.ContractError),  # fp32 path: bq power of two
    (dict(bf16=False, quant=True), sla2.ContractError),
    # fp32 path, bq = 256: one thread per query row holds d O columns and bk scores (<= 64 each)
    (dict(bf16=False, bq=256, bk=16, N=4096), sla2.ContractError),   # d = 128 columns
    (dict(bf16=False, bq=256, bk=128, d=16, N=4096), sla2.ContractError),  # 128 scores
])
def test_validation_errors(kw, err):
    base = dict(B=1, H=2, N=4096, d=128)
    base.update(kw)
    p = sla2.FwdParams(**{k: v for k, v in base.items() if k in ("B", "H", "N", "d")})
    for k, v in kw.items():
        setattr(p, k, v)
    with pytest.raises(err):
        sla2.workspace_bytes(p)


def test_f32_bq256_within_register_arrays_accepted():
    p = sla2.FwdParams(1, 1, 1024, 64, bq=256, bk=64, k_percent=25.0, bf16=False)
    assert sla2.workspace_bytes(p) > 0


def test_workspace_size_cfg2():
    n = sla2.workspace_bytes(sla2.FwdParams(1, 12, 32768, 128))
    # phi(K~) and phi(Q) bf16 (96 MiB each) dominate; everything else is O(B H (N/b) d)
    assert 192 * 2 ** 20 < n < 300 * 2 ** 20


def test_no_cpu_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    p = sla2.FwdParams(1, 1, 1024, 128).c()
    rc = sla2.lib().sla2_forward(C.byref(p), None, None, None, None, None, None, None, None, None, None, None, 0, None)
    assert rc == 4  # SLA2_CUDA_ERROR
    assert b"no CUDA device" in sla2.lib().sla2_last_error() or b"sm_100a" in sla2.lib().sla2_last_error()


def test_ragged_n_accepted_on_bf16_path():
    """bf16, non-QAT: N need not divide into blocks (ragged extension, tests/test_ragged.py)."""
    p = sla2.FwdParams(1, 2, 32760, 128)
    assert (p.tm, p.tn) == (256, 512)
    assert sla2.workspace_bytes(p) > 0
