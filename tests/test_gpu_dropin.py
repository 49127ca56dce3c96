"""The drop-in on the reference's own types (include/sla2_b200/reference_dropin.hpp): binaries
built by `make -C oracle dropin` from the UNMODIFIED reference headers (they exist where
/root/reference does and travel to the GPU box in oracle/_ref/).

* model_ref / model_b200: one step of the reference's toy DiT (model.hpp) with SLA2 attention in
  every head. model_b200 includes sla2_b200/sla2.hpp before sla2/model.hpp, so
  Tape::sla2_attention (tape.hpp:263-286) runs smooth_k, block_scores, hard_topk and
  sla2_forward_blockwise on the B200 (fp32 kernels, Matrix<double> rounded to float), and the
  reference's own sla2_backward consumes the drop-in's SLA2ForwardSaved. Routers must agree on
  every (layer, head); output, loss and gradients within 1e-4 relative (float vs double).
* test_shim_refmode: tests/cpp/test_shim.cpp (the reference's forward KATs) on the reference's
  types."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

pytestmark = pytest.mark.gpu


def _blocks(path):
    raw = open(path, "rb").read()
    out, off = [], 0
    while off < len(raw):
        n = int(np.frombuffer(raw, np.uint32, 1, off)[0])
        out.append(np.frombuffer(raw, np.float64, n, off + 4))
        off += 4 + 8 * n
    return out


def _need(name):
    p = os.path.join(REF, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (make -C oracle dropin needs /root/reference)")
    return p


@pytest.mark.parametrize("k_percent,seed", [(25.0, 7), (12.5, 3)])
def test_model_forward_through_dropin(cuda, tmp_path, k_percent, seed):
    ref_bin, b200_bin = _need("model_ref"), _need("model_b200")
    outs = {}
    for name, exe in (("ref", ref_bin), ("b200", b200_bin)):
        f = str(tmp_path / f"{name}.bin")
        r = subprocess.run([exe, f, str(k_percent), str(seed)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[name] = _blocks(f)
    ref, got = outs["ref"], outs["b200"]
    assert len(ref) == len(got) == 4 + 4  # out, loss, dw_in, dwq0, 2 layers x 2 heads of masks
    for h, (a, b) in enumerate(zip(ref[4:], got[4:])):
        assert np.array_equal(a, b), f"router mask differs (layer/head record {h})"
    for name, a, b in zip(("out", "loss", "dL/dw_in", "dL/dwq[0]"), ref[:4], got[:4]):
        e = np.abs(a - b).max() / max(np.abs(a).max(), 1e-30)
        assert e <= 1e-4, (name, e)


def test_shim_on_reference_types(cuda):
    exe = _need("test_shim_refmode")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
