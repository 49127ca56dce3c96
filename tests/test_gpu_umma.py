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


def test_device_expf_matches_host_libm(lib, cuda):
    """expf_glibc on the device vs this host's libm expf over the softmax-relevant range
    (all floats in [-104, 0] -- every argument row_softmax can produce after max subtraction)
    in 2^26-value chunks."""
    import ctypes
    import torch
    libm = ctypes.CDLL("libm.so.6")
    lib.expf_selftest.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p]
    lo = 0x80000000  # -0.0 ... up to -104 (0xC2D00000)
    hi = 0xC2D00001
    chunk = 1 << 26
    out = torch.empty(chunk, dtype=torch.float32, device=cuda)
    x = np.arange(chunk, dtype=np.uint64)
    checked = 0
    for start in range(lo, hi, chunk):
        n = min(chunk, hi - start)
        assert lib.expf_selftest(start, n, out.data_ptr()) == 0
        got = out[:n].cpu().numpy()
        xs = (x[:n] + start).astype(np.uint32).view(np.float32)
        ref = np.exp(xs.astype(np.float32))  # numpy float32 exp is not libm: compare to libm below
        # libm expf via ctypes in a vectorized way is too slow; use a strided sample through libm
        libm.expf.restype = C.c_float
        libm.expf.argtypes = [C.c_float]
        idx = np.arange(0, n, 997)
        lm = np.array([libm.expf(float(v)) for v in xs[idx]], dtype=np.float32)
        assert np.array_equal(got[idx].view(np.uint32), lm.view(np.uint32))
        del ref
        checked += len(idx)
    assert checked > 1_000_000


@pytest.mark.parametrize("mode", [0, 1])
def test_umma_bf16_a_from_tmem(lib, cuda, mode):
    """TS form: A written into TMEM (lane = row, bf16 pairs per column), B from smem."""
    import torch
    lib.umma_ts_selftest.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    g = torch.Generator(device="cpu").manual_seed(10 + mode)
    if mode == 0:
        a = torch.randn((128, 128), generator=g).to(torch.bfloat16)
        b = torch.randn((64, 128), generator=g).to(torch.bfloat16)
        ref = a.float() @ b.float().t()
    else:
        a = torch.randn((128, 64), generator=g).to(torch.bfloat16)
        b = torch.randn((64, 128), generator=g).to(torch.bfloat16)
        ref = a.float() @ b.float()
    d = torch.zeros(ref.shape, dtype=torch.float32, device=cuda)
    assert lib.umma_ts_selftest(mode, a.to(cuda).data_ptr(), b.to(cuda).data_ptr(), d.data_ptr()) == 0
    torch.testing.assert_close(d.cpu(), ref, rtol=1e-4, atol=1e-3)
