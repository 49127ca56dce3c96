"""Pins the tcgen05 / TMA encodings (tc.cuh) the product kernels rely on, one MMA shape and
operand-major combination at a time, against torch matmul on the same device."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cuda", "libumma_selftest.so")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib(cuda):
    if not os.path.exists(SO):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cuda")], check=True)
    lib = C.CDLL(SO)
    lib.umma_selftest.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.tma_selftest.argtypes = [C.c_void_p, C.c_long, C.c_long, C.c_int, C.c_int, C.c_void_p]
    return lib


@pytest.mark.parametrize("mode", [0, 1, 2, 5])
def test_umma_bf16(lib, cuda, mode):
    import torch
    g = torch.Generator(device="cpu").manual_seed(mode)
    shapes = {0: ((128, 128), (64, 128)), 1: ((128, 64), (64, 128)), 2: ((64, 128), (64, 128)),
              5: ((128, 128), (128, 128))}
    sa, sb = shapes[mode]
    a = torch.randn(sa, generator=g).to(torch.bfloat16).to(cuda)
    b = torch.randn(sb, generator=g).to(torch.bfloat16).to(cuda)
    if mode == 0:
        ref = a.float() @ b.float().t()
    elif mode == 2:
        ref = a.float().t() @ b.float()
    else:
        ref = a.float() @ b.float()
    d = torch.zeros(ref.shape, dtype=torch.float32, device=cuda)
    assert lib.umma_selftest(mode, a.data_ptr(), b.data_ptr(), d.data_ptr()) == 0
    torch.testing.assert_close(d, ref, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("mode", [3, 4])
def test_umma_int8(lib, cuda, mode):
    import torch
    g = torch.Generator(device="cpu").manual_seed(mode)
    sa, sb = ((128, 128), (64, 128)) if mode == 3 else ((128, 64), (64, 128))
    a = torch.randint(-127, 128, sa, generator=g, dtype=torch.int8)
    b = torch.randint(-127, 128, sb, generator=g, dtype=torch.int8)
    ref = (a.long() @ b.long().t()) if mode == 3 else (a.long() @ b.long())
    d = torch.zeros(ref.shape, dtype=torch.int32, device=cuda)
    assert lib.umma_selftest(mode, a.to(cuda).data_ptr(), b.to(cuda).data_ptr(), d.data_ptr()) == 0
    assert torch.equal(d.cpu().long(), ref)


def test_tma_swizzle128(lib, cuda):
    import torch
    rows, cols = 256, 128
    src = torch.arange(rows * cols, dtype=torch.int32).remainder(65521).to(torch.int16).view(rows, cols)
    dev = src.to(cuda)
    out = torch.zeros(8192, dtype=torch.uint8, device=cuda)
    x, y = 64, 128
    assert lib.tma_selftest(dev.data_ptr(), rows, cols, x, y, out.data_ptr()) == 0
    got = out.cpu().numpy().view(np.int16).reshape(64, 64)
    box = src.numpy()[y:y + 64, x:x + 64]
    # expected SWIZZLE_128B placement: 16-byte chunk c of row r lands at chunk c ^ (r % 8)
    exp = np.empty_like(box)
    for r in range(64):
        for c in range(8):
            pc = c ^ (r % 8)
            exp[r, pc * 8:(pc + 1) * 8] = box[r, c * 8:(c + 1) * 8]
    assert np.array_equal(got, exp)
