"""RTEN1 golden exchange (the reference's tensor_io.hpp:12-115).

CPU: paper_2602_12675_b200.rten1 reads what the reference's own writer (sla2::rten::save through
oracle/_ref) wrote, and the reference's own reader reads what it writes; the error paths raise
the reference's contract_error messages. GPU: the fixtures in tests/golden/rten1/ -- inputs and
outputs of one reference forward written by the reference itself (tests/golden/make_rten1.py)
-- drive the device forward, which must reproduce the reference's mask bit for bit and its
output within the bf16 tolerance."""
import os

import numpy as np
import pytest

import oracle_ctypes as oc
import paper_2602_12675_b200 as sla2
from paper_2602_12675_b200 import rten1

R = oc.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built (no /root/reference here)")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "rten1")


@pytest.mark.parametrize("shape,dtype", [((7, 5), np.float32), ((3, 4), np.float64), ((9,), np.float32),
                                         ((2, 3, 4), np.float64), ((0, 4), np.float32)])
def test_round_trip(tmp_path, shape, dtype):
    a = np.random.default_rng(1).standard_normal(shape).astype(dtype)
    f = tmp_path / "t.rten"
    rten1.save(f, a)
    b = rten1.load(f)
    assert b.dtype == dtype and b.shape == a.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    raw = f.read_bytes()
    assert raw[:6] == b"RTEN1\x00" and raw[6:10] == len(shape).to_bytes(4, "little")


@needs_ref
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_interop_with_reference(tmp_path, dtype):
    m = np.random.default_rng(2).standard_normal((6, 9)).astype(dtype)
    v = np.random.default_rng(3).standard_normal(11).astype(dtype)
    # reference writes -> we read
    R.rten_save(tmp_path / "m_ref.rten", m)
    R.rten_save(tmp_path / "v_ref.rten", v)
    assert np.array_equal(rten1.load_matrix(tmp_path / "m_ref.rten", dtype), m)
    assert np.array_equal(rten1.load_vector(tmp_path / "v_ref.rten", dtype), v)
    # we write -> reference reads
    rten1.save_matrix(tmp_path / "m_us.rten", m)
    rten1.save_vector(tmp_path / "v_us.rten", v)
    assert np.array_equal(R.rten_load(tmp_path / "m_us.rten", m.shape, dtype), m)
    assert np.array_equal(R.rten_load(tmp_path / "v_us.rten", v.shape, dtype), v)
    assert (tmp_path / "m_ref.rten").read_bytes() == (tmp_path / "m_us.rten").read_bytes()


def test_errors(tmp_path):
    f = tmp_path / "bad.rten"
    f.write_bytes(b"RTEN2\x00" + bytes(8))
    with pytest.raises(sla2.ContractError, match="bad magic"):
        rten1.load(f)
    rten1.save(f, np.zeros((2, 2), np.float64))
    with pytest.raises(sla2.ContractError, match="dtype mismatch"):
        rten1.load_matrix(f, np.float32)
    f.write_bytes(f.read_bytes()[:-3])
    with pytest.raises(sla2.ContractError, match="truncated"):
        rten1.load(f)
    rten1.save(f, np.zeros(3, np.float32))
    with pytest.raises(sla2.ContractError, match="expected rank 2"):
        rten1.load_matrix(f)
    with pytest.raises(sla2.ContractError, match="f32 and f64"):
        rten1.save(f, np.zeros(3, np.int32))


def _gold(name):
    return rten1.load(os.path.join(GOLD, f"wan_n256_{name}.rten"), np.float32)


@needs_ref
def test_fixtures_match_reference_now():
    """The committed fixtures are what the reference computes on their inputs (regenerable)."""
    q, k, v = _gold("q"), _gold("k"), _gold("v")
    out, mask, o_s, o_l, big_l = R.attention(q, k, v, 128, 64, _gold("proj_q"), _gold("proj_k"), _gold("rho"),
                                             float(_gold("k_percent")[0]))
    assert np.array_equal(out, _gold("out")) and np.array_equal(mask.astype(np.float32), _gold("mask"))


@pytest.mark.gpu
def test_gpu_forward_on_reference_rten1_goldens(cuda):
    import torch
    from sla2_testlib import rel_err
    q, k, v = (torch.from_numpy(_gold(n))[None, None].to(cuda, torch.bfloat16) for n in ("q", "k", "v"))
    pq, pk = (torch.from_numpy(_gold(n))[None].to(cuda) for n in ("proj_q", "proj_k"))
    rho = torch.from_numpy(_gold("rho"))[None].to(cuda)
    out, mask = sla2.forward(q, k, v, pq, pk, rho, k_percent=float(_gold("k_percent")[0]), return_mask=True)
    assert np.array_equal(mask.cpu().numpy()[0, 0].astype(np.float32), _gold("mask"))
    assert rel_err(out.float().cpu().numpy()[0, 0], _gold("out"))[0] <= 1e-2
