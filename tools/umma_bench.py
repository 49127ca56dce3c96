"""Cycles per tcgen05.mma (M=128, bf16): issue variants x operand forms x N; one CTA per SM."""
import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = C.CDLL(os.path.join(HERE, "..", "tests", "cuda", "libumma_bench.so"))
L.umma_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
forms = {0: "SS K/K  ", 1: "SS K/MN ", 2: "SS MN/MN", 3: "TS B-K  ", 4: "TS B-MN "}
variants = {0: "lane0 loop", 1: "lane0 unroll8", 2: "warp elect x8", 3: "elect 2 acc", 4: "elect 4 acc",
            5: "fresh addr"}
cyc = torch.zeros(148, dtype=torch.int64, device="cuda")
gbuf = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
reps = 1024
for form in (0, 1, 2, 3, 4):
    for n in (64, 128, 256):
        row = []
        for v in range(6):
            if v == 3 and n > 128:
                row.append("   -  ")
                continue
            if v == 4 and n > 64:
                row.append("   -  ")
                continue
            assert L.umma_bench(form, v, n, reps, 148, cyc.data_ptr(), gbuf.data_ptr()) == 0
            row.append(f"{cyc.float().mean().item() / reps:6.1f}")
        print(f"{forms[form]} N={n:3d} ideal {128 * n / 256:5.1f} | " + " | ".join(
            f"{variants[v]}: {row[v]}" for v in range(6)))
reps = 1032  # multiple of 24
for v, name in ((6, "PV x8, QK x8, HS x8"), (7, "same, QK overwrites P cols"), (8, "PV x8, HS x8 (per 24)"),
                (9, "6 + commit per group"), (10, "9 + try_wait + fence::after per group")):
    for fl, fname in ((0, ""), (16, " +TMEM ld/st"), (32, " +bulk copies"), (48, " +both")):
        assert L.umma_bench(0, v + fl, 128, reps, 148, cyc.data_ptr(), gbuf.data_ptr()) == 0
        c = cyc.float().mean().item() / reps
        print(f"pair mix [{name}{fname}]: {c:6.1f} cycles/MMA (ideal 64)")
