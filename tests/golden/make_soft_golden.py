"""Writes tests/golden/soft_*.npz with the UNMODIFIED reference (oracle/_ref): the stage-1 soft
routing chain of stage1_record_grads (training.hpp:186-201) -- pc = block_scores(Q, smooth_k(K))
(router.hpp:87-102), soft_topk (router.hpp:126-190) and sla2_forward_blockwise with the SoftMask
(attention.hpp:484-558) -- in float, so the device path is checked where oracle/_ref is absent.
Run where /root/reference exists."""
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
    for name, n, d, bq, bk, kp, tau, seed in (("soft_n256_d64", 256, 64, 64, 64, 50.0, 0.1, 81),
                                               ("soft_n512_d32_bq32", 512, 32, 32, 64, 25.0, 0.05, 82)):
        q, k, v, pq, pk, rho = make_inputs(1, 1, n, d, seed, bf16=False, bq=bq, bk=bk)
        q, k, v, pq, pk, rho = q[0, 0], k[0, 0], v[0, 0], pq[0], pk[0], rho[0]
        kt, _ = R.smooth_k(k)
        pc = R.block_scores(q, kt, pq, pk, bq, bk, tau)
        values, lambdas = R.soft_topk(pc, kp, tau)
        out, o_s, o_l, big_l = R.forward_soft(q, k, v, bq, bk, values, rho)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), q=q, k=k, v=v, proj_q=pq, proj_k=pk, rho=rho,
                            bq=bq, bk=bk, k_percent=kp, tau=np.float32(tau), pc=pc, values=values,
                            lambdas=lambdas, out=out, o_s=o_s, o_l=o_l, big_l=big_l)
        print(name, float(np.abs(out).max()), float(values.sum()))


if __name__ == "__main__":
    main()
