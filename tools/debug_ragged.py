"""Analysis only: locate the first ragged-N stage that departs from the oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2602_12675_b200 as sla2
import oracle_ctypes as oc
from test_ragged import _gpu_case
from sla2_testlib import to_dev
P = oc.port()
dev = torch.device("cuda:0")
for N in (4000, 1000):
    q, k, v, pq, pk, rho = _gpu_case(1, 1, N, 1)
    kt, mu = P.smooth_k(k[0, 0])
    _, gmu = sla2.smooth_k(to_dev(k, torch.bfloat16, dev))
    gm = gmu.float().cpu().numpy().reshape(-1)[:128]
    print(N, "mu equal:", np.array_equal(gm.view(np.uint32), mu.view(np.uint32)), np.abs(gm - mu).max())
    tm, tn = -(-N // 128), -(-N // 64)
    pc = np.empty((tm, tn), np.float32)
    assert P._block_scores_ragged_f(q[0, 0], kt, N, 128, pq[0], pk[0], np.float32(0.1), 128, 64, pc) == 0
    gpc, gmask, gidx = sla2.router(to_dev(q, torch.bfloat16, dev), to_dev(k, torch.bfloat16, dev),
                                   to_dev(pq, torch.float32, dev), to_dev(pk, torch.float32, dev), k_percent=5.0)
    gpc = gpc.cpu().numpy()[0, 0]
    bad = np.argwhere(gpc.view(np.uint32) != pc.view(np.uint32))
    print(N, "pc mismatches:", len(bad), bad[:5], "max", np.abs(gpc - pc).max())
    if len(bad):
        r, c = bad[0]
        print("  row", r, "col", c, gpc[r, c], pc[r, c], "last row/col:", tm - 1, tn - 1)
