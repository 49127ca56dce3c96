"""Writes tests/golden/backward_*.npz with the UNMODIFIED reference (oracle/_ref): inputs, the
reference's routing mask and its sla2_backward gradients (attention.hpp:610-809), so the device
backward can be checked where oracle/_ref is absent. Run where /root/reference exists."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_ctypes as oc  # noqa: E402
from sla2_testlib import make_inputs  # noqa: E402


def main():
    R = oc.ref()
    assert R is not None, "build oracle/_ref first (make -C oracle)"
    for name, n, d, bq, bk, kp, seed in (("backward_n256_d64", 256, 64, 64, 64, 50.0, 61),
                                          ("backward_n512_d32_bq32", 512, 32, 32, 64, 25.0, 62)):
        q, k, v, pq, pk, rho = make_inputs(1, 1, n, d, seed, bf16=False, bq=bq, bk=bk)
        q, k, v, pq, pk, rho = q[0, 0], k[0, 0], v[0, 0], pq[0], pk[0], rho[0]
        d_out = np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)
        mask = R.attention(q, k, v, bq, bk, pq, pk, rho, kp)[1]
        dq, dk, dv, drho = R.backward(q, k, v, bq, bk, mask, rho, d_out)[:4]
        np.savez_compressed(os.path.join(HERE, name + ".npz"), q=q, k=k, v=v, proj_q=pq, proj_k=pk, rho=rho,
                            bq=bq, bk=bk, k_percent=kp, d_out=d_out, mask=mask, dq=dq, dk=dk, dv=dv, drho=drho)
        print(name, float(np.abs(dq).max()), int(mask.sum()))


if __name__ == "__main__":
    main()
