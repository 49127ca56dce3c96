"""Generates tests/golden/*.npz by running the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj/include by oracle/Makefile) on seeded inputs. Run once in a container that
has /root/reference; the fixtures let the oracle and the GPU path be checked on machines
without it (the GPU box). Inputs use the reference's own test streams (test_util.hpp) where
the reference tests do, and bf16-valued floats for the GPU block shape."""
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
    cases = []
    # the reference's blockwise-vs-naive case (test_attention.cpp:215-241), random_inputs streams
    for dt in (np.float64, np.float32):
        for seed, kp in ((351, 10.0), (352, 25.0), (353, 50.0)):
            q, k, v = (R.gaussian((64, 8), seed + i, dtype=dt) for i in range(3))
            cases.append((f"ref_tests_n64_d8_s{seed}_{np.dtype(dt).name}", q, k, v, 8, 4,
                          np.eye(8, dtype=dt), np.eye(8, dtype=dt), np.zeros(8, dt), kp, False))
    # QAT on the reference test shape
    q, k, v = (R.gaussian((32, 8), 363 + i, dtype=np.float32) for i in range(3))
    cases.append(("ref_tests_qat_n32_d8", q, k, v, 4, 4, np.eye(8, dtype=np.float32), np.eye(8, dtype=np.float32),
                  np.zeros(8, np.float32), 25.0, True))
    # the GPU block shape (d = 128, bq = 128, bk = 64) on bf16-valued inputs, bf16 + QAT
    for seed, kp, quant in ((5, 25.0, False), (6, 40.0, False), (7, 25.0, True)):
        qb, kb, vb, pq, pk, rho = make_inputs(1, 1, 512, 128, seed=seed)
        cases.append((f"wan_blocks_n512_s{seed}{'_qat' if quant else ''}", qb[0, 0], kb[0, 0], vb[0, 0], 128, 64,
                      pq[0], pk[0], rho[0], kp, quant))
    # fp32 config-1 geometry, smaller N
    q1, k1, v1, pq1, pk1, rho1 = make_inputs(1, 1, 512, 64, seed=9, bf16=False, bq=64, bk=64)
    cases.append(("cfg1_blocks_n512", q1[0, 0], k1[0, 0], v1[0, 0], 64, 64, pq1[0], pk1[0], rho1[0], 10.0, False))
    for name, q, k, v, bq, bk, pq, pk, rho, kp, quant in cases:
        out, mask, o_s, o_l, big_l = R.attention(q, k, v, bq, bk, pq, pk, rho, kp, quant=quant)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), q=q, k=k, v=v, bq=bq, bk=bk, proj_q=pq, proj_k=pk,
                            rho=rho, k_percent=kp, quant=quant, out=out, mask=mask, o_s=o_s, o_l=o_l, big_l=big_l)
        print(name, out.dtype, mask.sum())


if __name__ == "__main__":
    main()
