"""Writes tests/golden/rten1/*.rten with the UNMODIFIED reference's own RTEN1 writer
(sla2::rten::save, tensor_io.hpp) through oracle/_ref: the inputs and the reference's outputs of
one Tape::sla2_attention forward at the GPU block shape (d = 128, bq = 128, bk = 64) on
bf16-valued inputs. The GPU harness reads them with paper_2602_12675_b200.rten1 (SURVEY.md 8f
item 4: golden exchange between the GPU harness and the oracle). Run where /root/reference is
available (make -C oracle first)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_ctypes as oc  # noqa: E402
from sla2_testlib import make_inputs  # noqa: E402

OUT = os.path.join(HERE, "rten1")


def main():
    R = oc.ref()
    assert R is not None, "build oracle/_ref first (make -C oracle)"
    os.makedirs(OUT, exist_ok=True)
    n, d, bq, bk, kp = 256, 128, 128, 64, 50.0
    q, k, v, pq, pk, rho = make_inputs(1, 1, n, d, seed=31)
    q, k, v, pq, pk, rho = q[0, 0], k[0, 0], v[0, 0], pq[0], pk[0], rho[0]
    out, mask, o_s, o_l, big_l = R.attention(q, k, v, bq, bk, pq, pk, rho, kp)
    tensors = dict(q=q, k=k, v=v, proj_q=pq, proj_k=pk, rho=rho, out=out, o_s=o_s, o_l=o_l, big_l=big_l,
                   mask=mask.astype(np.float32), k_percent=np.array([kp], np.float32))
    for name, a in tensors.items():
        R.rten_save(os.path.join(OUT, f"wan_n256_{name}.rten"), np.ascontiguousarray(a, np.float32))
        print(name, a.shape)


if __name__ == "__main__":
    main()
