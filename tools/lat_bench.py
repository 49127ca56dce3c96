"""Dependent-chain latency of the exact column mean's add (analysis only)."""
import ctypes as C
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = C.CDLL(os.path.join(HERE, "..", "tests", "cuda", "liblat_bench.so"))
L.lat_bench.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p]
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
out = torch.zeros(32, dtype=torch.float32, device="cuda")
n = 4096
for w, name in ((0, "FADD f32+f32"), (1, "FHADD f32+bf16 (reg)"), (2, "LDS.U16 -> FHADD (chain + loads)"),
                (3, "LDS.32 -> 2 FHADD chains (per row)"), (4, "LDS.64 -> 4 FHADD chains (per row)")):
    for _ in range(2):
        assert L.lat_bench(w, n, cyc.data_ptr(), out.data_ptr()) == 0
    print(f"{name:34s} {cyc.item() / n:6.2f} cycles/op")
