"""paper_2602_12675_b200 -- B200-native (sm_100a) SLA2 forward pass behind the reference's API.

Python mirror of the reference's C++ operator interface for the SLA2 hot path
(/root/reference/proj/include/sla2), calling libsla2_b200.so through its C ABI
(include/sla2_capi.h). Names, argument meaning and error classes follow the reference:

  smooth_k(k)                                   quant.hpp:88-96
  block_scores(q, k, proj_q, proj_k, bq, bk)    router.hpp:87-102
  hard_topk(pc, k_percent)                      router.hpp:106-125
  topk_budget(k_percent, tn)                    router.hpp:36-40
  sla2_forward_blockwise(q, k, v, mask, rho)    attention.hpp:423-560
  sla2_attention(q, k, v, rho, proj, ...)       tape.hpp:263-272 (router + forward)
  full_attention(q, k, v)                       attention.hpp:71-75 (dense tcgen05 baseline)

Tensors are torch CUDA tensors shaped [B, H, N, d] (each [b, h] slice is one reference
Matrix), bf16 or fp32; per-head router state is proj [H, d, d] fp32 and rho [H, tm] fp32.
Errors raise ShapeError / NumericError / ContractError (sla2::shape_error, numeric_error,
contract_error of common.hpp:13-29) or CudaError. There is no CPU fallback: without the built
library or an sm_100a GPU every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

__all__ = [
    "ShapeError", "NumericError", "ContractError", "CudaError", "Sla2Error",
    "lib", "library_path", "topk_budget", "smooth_k", "quantize", "linear_precompute", "block_scores", "hard_topk",
    "sla2_forward_blockwise", "sla2_attention", "full_attention", "router", "forward",
    "FwdParams", "workspace_bytes", "last_launch_count",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("SLA2_LIB") or os.path.join(_HERE, "libsla2_b200.so")  # SLA2_LIB: analysis builds


class Sla2Error(RuntimeError):
    pass


class ShapeError(Sla2Error, ValueError):
    """sla2::shape_error (common.hpp:14-17)."""


class NumericError(Sla2Error):
    """sla2::numeric_error (common.hpp:20-23)."""


class ContractError(Sla2Error):
    """sla2::contract_error (common.hpp:26-29)."""


class CudaError(Sla2Error):
    """Launch failure or no sm_100a device (no CPU fallback exists)."""


class _Params(C.Structure):
    _fields_ = [("B", C.c_int64), ("H", C.c_int64), ("N", C.c_int64), ("d", C.c_int64),
                ("bq", C.c_int64), ("bk", C.c_int64), ("k_percent", C.c_double),
                ("dtype", C.c_int32), ("quant", C.c_int32), ("smooth", C.c_int32),
                ("exact_mu", C.c_int32), ("tau", C.c_float), ("reserved", C.c_int32 * 3)]


class _Saved(C.Structure):
    _fields_ = [("o_s", C.c_void_p), ("o_l", C.c_void_p), ("big_l", C.c_void_p), ("h_blocks", C.c_void_p),
                ("z_blocks", C.c_void_p), ("q_phi", C.c_void_p), ("k_phi", C.c_void_p),
                ("qat_s_first", C.c_void_p)]


def _saved_buffers(p, q, full, qat_s):
    """Device buffers for SLA2ForwardSaved (attention.hpp:345-358): o_s, o_l, big_l; with full=True
    also h_blocks [B,H,tm,d,d], z_blocks [B,H,tm,d], q_phi, k_phi [B,H,N,d]; qat_s: the QAT S hook."""
    import torch
    dev = q.device
    f32 = dict(dtype=torch.float32, device=dev)
    svs = {"o_s": torch.empty(q.shape, **f32), "o_l": torch.empty(q.shape, **f32), "big_l": torch.empty(q.shape[:3], **f32)}
    if full:
        svs["h_blocks"] = torch.empty((p.B, p.H, p.tm, p.d, p.d), **f32)
        svs["z_blocks"] = torch.empty((p.B, p.H, p.tm, p.d), **f32)
        svs["q_phi"] = torch.empty(q.shape, **f32)
        svs["k_phi"] = torch.empty(q.shape, **f32)
    if qat_s:
        svs["qat_s_first"] = torch.empty((p.B, p.H, p.tm, p.bq, p.bk), **f32)
    sv = _Saved(*[svs[n].data_ptr() if n in svs else None for n, _ in _Saved._fields_])
    return sv, svs


_lib = None


def library_path() -> str:
    return _SO


def lib():
    """Load libsla2_b200.so (built by __graft_entry__.build() / make). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise CudaError(f"{_SO} is not built (run python -c 'import __graft_entry__ as g; g.build()');"
                        " there is no CPU fallback")
    L = C.CDLL(_SO)
    vp, sz, P = C.c_void_p, C.c_size_t, C.POINTER(_Params)
    sig = {
        "sla2_default_params": ([P, C.c_int64, C.c_int64, C.c_int64, C.c_int64], None),
        "sla2_topk_budget": ([C.c_double, C.c_int64], C.c_int64),
        "sla2_check_params": ([P], C.c_int),
        "sla2_workspace_size": ([P], sz),
        "sla2_forward": ([P, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(_Saved), vp, sz, vp], C.c_int),
        "sla2_router": ([P, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_smooth_k": ([P, vp, vp, vp, vp], C.c_int),
        "sla2_hard_topk": ([P, vp, vp, vp, vp], C.c_int),
        "sla2_quantize": ([P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_linear_precompute": ([P, vp, vp, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_sparse_fwd": ([P, vp, vp, vp, vp, vp, vp, C.POINTER(_Saved), vp, sz, vp], C.c_int),
        "sla2_dense_fwd": ([P, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_forward_host": ([P, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "sla2_backward_workspace_size": ([P], sz),
        "sla2_soft_topk": ([P, vp, vp, vp, vp], C.c_int),
        "sla2_forward_soft_workspace_size": ([P], sz),
        "sla2_soft_topk_backward": ([P, vp, vp, vp, vp], C.c_int),
        "sla2_forward_soft": ([P, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_backward": ([P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp], C.c_int),
        "sla2_last_error": ([], C.c_char_p),
        "sla2_last_launch_count": ([], C.c_int32),
        "sla2_version": ([], C.c_char_p),
        "sla2_enable_stage_timing": ([C.c_int32], None),
        "sla2_last_stage_ms": ([C.POINTER(C.c_float), C.c_int32], C.c_int32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _raise(rc: int):
    if rc == 0:
        return
    msg = lib().sla2_last_error().decode()
    cls = {1: ShapeError, 2: NumericError, 3: ContractError}.get(rc, CudaError)
    raise cls(msg)


def last_launch_count() -> int:
    """Kernel launches enqueued by the last call on this thread."""
    return int(lib().sla2_last_launch_count())


def enable_stage_timing(on: bool = True):
    lib().sla2_enable_stage_timing(1 if on else 0)


def last_stage_ms(timeline=False):
    """(router, linear precompute, sparse kernel, total) ms of the last forward (CUDA events);
    with timeline=True also (mu ready, query side done, key prep done, router back done,
    linear precompute done), ms since the call started (-1: not on this path)."""
    buf = (C.c_float * 9)()
    n = lib().sla2_last_stage_ms(buf, 9 if timeline else 4)
    return tuple(float(buf[i]) for i in range(n))


def topk_budget(k_percent: float, tn: int) -> int:
    """router.hpp:36-40: kappa = min(tn, max(1, llround(k%/100 * tn)))."""
    return int(lib().sla2_topk_budget(float(k_percent), int(tn)))


@dataclass
class FwdParams:
    B: int
    H: int
    N: int
    d: int
    bq: int = 128
    bk: int = 64
    k_percent: float = 3.0
    bf16: bool = True
    quant: bool = False
    smooth: bool = True
    exact_mu: bool = True
    tau: float = 0.1

    def c(self) -> _Params:
        p = _Params()
        p.B, p.H, p.N, p.d, p.bq, p.bk = self.B, self.H, self.N, self.d, self.bq, self.bk
        p.k_percent = float(self.k_percent)
        p.dtype = 1 if self.bf16 else 0
        p.quant = _quant_code(self.quant)
        p.smooth = int(bool(self.smooth))
        p.exact_mu = int(bool(self.exact_mu))
        p.tau = float(self.tau)
        return p

    @property
    def tm(self):
        return -(-self.N // self.bq)  # ceil: a ragged N has a partial last block (bf16 path)

    @property
    def tn(self):
        return -(-self.N // self.bk)

    @property
    def kappa(self):
        return topk_budget(self.k_percent, self.tn)


def workspace_bytes(p: FwdParams) -> int:
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    return int(lib().sla2_workspace_size(C.byref(cp)))


_ws_cache = {}


def _workspace(p: FwdParams, device):
    import torch
    n = workspace_bytes(p)
    key = (device.index if device.index is not None else 0)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 1), dtype=torch.uint8, device=device)
        _ws_cache[key] = buf
    return buf


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(dev):
    import torch
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _quant_code(quant) -> int:
    """quant: False / "none" -> SLA2_QUANT_NONE; True / "int8" -> SLA2_QUANT_INT8 (the reference's
    QuantConfig, quant.hpp:15-19, reproduced exactly); "fp8" -> SLA2_QUANT_FP8PV (E4M3 P / V,
    tolerance only; not a reference mode)."""
    if isinstance(quant, str):
        codes = {"none": 0, "int8": 1, "fp8": 2}
        if quant not in codes:
            raise ContractError(f"unknown quant mode {quant!r} (none, int8, fp8)")
        return codes[quant]
    return 1 if quant else 0


def _params_from(q, bq, bk, k_percent, quant, smooth, exact_mu, tau=0.1):
    import torch
    if q.dim() != 4:
        raise ShapeError("expected [B, H, N, d] tensors")
    if q.dtype not in (torch.bfloat16, torch.float32):
        raise ContractError("q/k/v must be bfloat16 or float32")
    B, H, N, d = q.shape
    return FwdParams(B, H, N, d, bq, bk, k_percent, q.dtype == torch.bfloat16, quant, smooth, exact_mu, tau)


def _check_like(ref, *ts):
    for t in ts:
        if t.shape != ref.shape or t.dtype != ref.dtype or t.device != ref.device:
            raise ShapeError("AttentionInputs: q, k, v must share N x d")  # attention.hpp:36-38
        if not t.is_contiguous():
            raise ContractError("tensors must be contiguous")


def forward(q, k, v, proj_q, proj_k, rho, *, k_percent=3.0, bq=128, bk=64, quant=False, smooth=True,
            exact_mu=True, return_mask=False, return_idx=False, saved=False, out=None, workspace=None):
    """Router + blockwise forward (tape.hpp:263-272). Returns out or a tuple with
    (mask [B,H,tm,tn] u8, idx [B,H,tm,kappa] i32, saved dict) as requested; saved=True gives
    o_s, o_l, big_l, saved="full" all of SLA2ForwardSaved (+ the QAT S hook). `workspace` (a
    uint8 CUDA tensor of at least workspace_bytes(...)) replaces the shared per-device cache.
    quant: False / "none"; True / "int8" (the reference's QuantConfig, exact codes); "fp8" (E4M3
    P / V on kind::f8f6f4, out only, tolerance per DESIGN.md 4.2; not a reference mode)."""
    import torch
    _check_like(q, k, v)
    p = _params_from(q, bq, bk, k_percent, quant, smooth, exact_mu)
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    dev = q.device
    out = torch.empty_like(q) if out is None else out
    mask = torch.empty((p.B, p.H, p.tm, p.tn), dtype=torch.uint8, device=dev) if return_mask else None
    idx = torch.empty((p.B, p.H, p.tm, p.kappa), dtype=torch.int32, device=dev) if return_idx else None
    sv = None
    svs = None
    if saved:
        sv, svs = _saved_buffers(p, q, saved == "full", _quant_code(quant) == 1 and saved == "full")
    if workspace is not None:
        if workspace.dtype != torch.uint8 or workspace.device != dev or workspace.numel() < workspace_bytes(p):
            raise ContractError("workspace too small (see workspace_bytes)")
        ws = workspace
    else:
        ws = _workspace(p, dev)
    rc = lib().sla2_forward(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(proj_q.contiguous()),
                            _ptr(proj_k.contiguous()), _ptr(rho.contiguous()), _ptr(out), _ptr(mask), _ptr(idx),
                            C.byref(sv) if sv is not None else None, _ptr(ws), ws.numel(), _stream(dev))
    _raise(rc)
    res = [out]
    if return_mask:
        res.append(mask)
    if return_idx:
        res.append(idx)
    if saved:
        res.append(svs)
    return res[0] if len(res) == 1 else tuple(res)


class CapturedForward:
    """forward() captured once into a CUDA graph and replayed: one graph launch per call instead
    of ~10 kernel launches, event records and host-side checks (the call is launch-bound at
    small shapes and pays ~20 us of host time at cfg2). The input / output tensors are fixed at
    capture; write new inputs into them (copy_) between replays. The graph owns its workspace
    for its lifetime (a later forward() needing a bigger shared workspace cannot free it)."""

    def __init__(self, q, k, v, proj_q, proj_k, rho, **kw):
        import torch
        self.out = kw.pop("out", None)
        if self.out is None:
            self.out = torch.empty_like(q)
        self.args = (q, k, v, proj_q, proj_k, rho)
        p = _params_from(q, kw.get("bq", 128), kw.get("bk", 64), kw.get("k_percent", 3.0), kw.get("quant", False),
                         kw.get("smooth", True), kw.get("exact_mu", True))
        self.workspace = torch.empty(max(workspace_bytes(p), 1), dtype=torch.uint8, device=q.device)
        kw["workspace"] = self.workspace
        self.kw = kw
        forward(*self.args, out=self.out, **kw)  # warm-up: streams, events, attributes, maps
        torch.cuda.synchronize(q.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            forward(*self.args, out=self.out, **kw)
        self.launches = last_launch_count()

    def __call__(self):
        self.graph.replay()
        return self.out


def forward_host(q, k, v, proj_q, proj_k, rho, *, k_percent=3.0, bq=128, bk=64, quant=False, smooth=True,
                 exact_mu=True, return_mask=False):
    """The reference's call shape: host (CPU) tensors in, host tensors out, through
    sla2_forward_host (copies pipelined per head against the compute). Pin the inputs
    (tensor.pin_memory()) for asynchronous copies."""
    import torch
    _check_like(q, k, v)
    if q.device.type != "cpu":
        raise ContractError("forward_host takes host tensors")
    p = _params_from(q, bq, bk, k_percent, quant, smooth, exact_mu)
    cp = p.c()
    out = torch.empty_like(q, pin_memory=q.is_pinned())
    mask = torch.empty((p.B, p.H, p.tm, p.tn), dtype=torch.uint8, pin_memory=q.is_pinned()) if return_mask else None
    rc = lib().sla2_forward_host(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(proj_q.contiguous()),
                                 _ptr(proj_k.contiguous()), _ptr(rho.contiguous()), _ptr(out), _ptr(mask))
    _raise(rc)
    return (out, mask) if return_mask else out


def router(q, k, proj_q, proj_k, *, k_percent=3.0, bq=128, bk=64, smooth=True, exact_mu=True, tau=0.1,
           return_pc=True):
    """smooth_k + block_scores + hard_topk on device -> (pc fp32, mask u8, idx i32)."""
    import torch
    _check_like(q, k)
    p = _params_from(q, bq, bk, k_percent, False, smooth, exact_mu, tau)
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    dev = q.device
    pc = torch.empty((p.B, p.H, p.tm, p.tn), dtype=torch.float32, device=dev) if return_pc else None
    mask = torch.empty((p.B, p.H, p.tm, p.tn), dtype=torch.uint8, device=dev)
    idx = torch.empty((p.B, p.H, p.tm, p.kappa), dtype=torch.int32, device=dev)
    ws = _workspace(p, dev)
    _raise(lib().sla2_router(C.byref(cp), _ptr(q), _ptr(k), _ptr(proj_q.contiguous()), _ptr(proj_k.contiguous()),
                             _ptr(pc), _ptr(mask), _ptr(idx), _ptr(ws), ws.numel(), _stream(dev)))
    return pc, mask, idx


def quantize(q, k, v, *, bq=128, bk=64, smooth=True):
    """The QAT operand quantization (quantize, quant.hpp:31-50) of every query block of Q and key
    block of K~ = K - colmean(K) and V, on device: returns {"q_codes", "k_codes", "v_codes" int8
    [B,H,N,d], "q_scales" fp32 [B,H,tm], "k_scales", "v_scales" fp32 [B,H,tn]}, bit-exact."""
    import torch
    _check_like(q, k, v)
    p = _params_from(q, bq, bk, 3.0, True, smooth, True)
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    dev = q.device
    res = {"q_codes": torch.empty(q.shape, dtype=torch.int8, device=dev),
           "k_codes": torch.empty(q.shape, dtype=torch.int8, device=dev),
           "v_codes": torch.empty(q.shape, dtype=torch.int8, device=dev),
           "q_scales": torch.empty((p.B, p.H, p.tm), dtype=torch.float32, device=dev),
           "k_scales": torch.empty((p.B, p.H, p.tn), dtype=torch.float32, device=dev),
           "v_scales": torch.empty((p.B, p.H, p.tn), dtype=torch.float32, device=dev)}
    ws = _workspace(p, dev)
    _raise(lib().sla2_quantize(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(res["q_codes"]), _ptr(res["q_scales"]),
                               _ptr(res["k_codes"]), _ptr(res["k_scales"]), _ptr(res["v_codes"]),
                               _ptr(res["v_scales"]), _ptr(ws), ws.numel(), _stream(dev)))
    return res


def linear_precompute(k, v, *, bq=128, bk=64, smooth=True):
    """The linear branch's key-side precompute (attention.hpp:456-475) on device: returns
    {"k_phi" [B,H,N,d] (exact row softmax of K~), "z_blocks" [B,H,tn,d] (z_j per key block),
    "h_total" [B,H,d,d] (sum_j phi(K~_j)^T V_j), "z_total" [B,H,d]}, fp32."""
    import torch
    _check_like(k, v)
    p = _params_from(k, bq, bk, 3.0, False, smooth, True)
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    dev = k.device
    f32 = dict(dtype=torch.float32, device=dev)
    res = {"k_phi": torch.empty(k.shape, **f32), "z_blocks": torch.empty((p.B, p.H, p.tn, p.d), **f32),
           "h_total": torch.empty((p.B, p.H, p.d, p.d), **f32), "z_total": torch.empty((p.B, p.H, p.d), **f32)}
    ws = _workspace(p, dev)
    _raise(lib().sla2_linear_precompute(C.byref(cp), _ptr(k), _ptr(v), _ptr(res["k_phi"]), _ptr(res["z_blocks"]),
                                        _ptr(res["h_total"]), _ptr(res["z_total"]), _ptr(ws), ws.numel(),
                                        _stream(dev)))
    return res


def smooth_k(k):
    """quant.hpp:88-96 on device: returns (K - mu as fp32, mu [B,H,d] fp32)."""
    import torch
    p = _params_from(k, 1, 1, 100.0, False, True, True)
    cp = p.c()
    mu = torch.empty((p.B, p.H, p.d), dtype=torch.float32, device=k.device)
    _raise(lib().sla2_smooth_k(C.byref(cp), _ptr(k.contiguous()), _ptr(mu), None, _stream(k.device)))
    return k.float() - mu[:, :, None, :], mu


def block_scores(q, k, proj_q, proj_k, bq, bk, tau=0.1):
    """router.hpp:87-102 (k is the already-smoothed K~ as the reference's callers pass it)."""
    pc, _, _ = router(q, k, proj_q, proj_k, k_percent=100.0, bq=bq, bk=bk, smooth=False, tau=tau)
    return pc


def hard_topk(pc, k_percent):
    """router.hpp:106-125 on a device score tensor [B,H,tm,tn] -> (mask u8, idx i32, kappa)."""
    import torch
    if pc.dim() != 4 or pc.dtype != torch.float32:
        raise ShapeError("pc must be [B, H, tm, tn] float32")
    B, H, tm, tn = pc.shape
    if not (0.0 < k_percent <= 100.0):
        raise ShapeError("hard_topk: k_percent must be in (0, 100]")
    # score-matrix geometry through the params struct: rows N/bq = tm, columns N/bk = tn
    cp = _Params()
    cp.B, cp.H, cp.N, cp.d, cp.bq, cp.bk = B, H, tm * tn, 1, tn, tm
    cp.k_percent, cp.dtype, cp.quant, cp.smooth, cp.exact_mu, cp.tau = k_percent, 0, 0, 1, 1, 0.1
    kappa = topk_budget(k_percent, tn)
    mask = torch.empty((B, H, tm, tn), dtype=torch.uint8, device=pc.device)
    idx = torch.empty((B, H, tm, kappa), dtype=torch.int32, device=pc.device)
    _raise(lib().sla2_hard_topk(C.byref(cp), _ptr(pc.contiguous()), _ptr(mask), _ptr(idx), _stream(pc.device)))
    return mask, idx, kappa


def sla2_forward_blockwise(q, k, v, mask, rho, *, bq=128, bk=64, quant=False, smooth=True, saved=False):
    """attention.hpp:423-560 with a caller-given BlockMask [B,H,tm,tn] (device u8)."""
    import torch
    _check_like(q, k, v)
    p = _params_from(q, bq, bk, 100.0, quant, smooth, True)
    cp = p.c()
    _raise(lib().sla2_check_params(C.byref(cp)))
    if tuple(mask.shape) != (p.B, p.H, p.tm, p.tn):
        raise ShapeError("sla2_forward_blockwise: mask geometry mismatch")  # attention.hpp:436-438
    dev = q.device
    out = torch.empty_like(q)
    sv = None
    svs = None
    if saved:
        sv, svs = _saved_buffers(p, q, saved == "full", _quant_code(quant) == 1 and saved == "full")
    ws = _workspace(p, dev)
    _raise(lib().sla2_sparse_fwd(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(rho.contiguous()),
                                 _ptr(mask.contiguous().to(torch.uint8)), _ptr(out),
                                 C.byref(sv) if sv is not None else None, _ptr(ws), ws.numel(), _stream(dev)))
    return (out, svs) if saved else out


def sla2_backward(q, k, v, d_out, rho, mask, saved, *, bq=64, bk=64, smooth=True):
    """attention.hpp:610-809 with hard routing (the stage-2 / QAT fine-tuning backward), on the
    device: fp32 q, k, v, d_out [B,H,N,d]; mask [B,H,tm,tn] u8 (the forward's routing); rho
    [H,tm]; `saved` = the dict forward(..., saved=True) returns (o_s, o_l, big_l). Returns
    {"dq", "dk", "dv", "drho" [B,H,tm]}. Full precision whatever the forward was."""
    import torch
    _check_like(q, k, v, d_out)
    if q.dtype != torch.float32:
        raise ContractError("sla2_backward: fp32 tensors (the backward is full precision)")
    p = _params_from(q, bq, bk, 100.0, False, smooth, True)
    cp = p.c()
    n = int(lib().sla2_backward_workspace_size(C.byref(cp)))
    if n == 0:
        _raise(lib().sla2_backward(C.byref(cp), *([None] * 14), 0, None))  # raises the validation error
    dev = q.device
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    drho = torch.empty((p.B, p.H, p.tm), dtype=torch.float32, device=dev)
    rc = lib().sla2_backward(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(rho.contiguous()), _ptr(mask.contiguous()),
                             _ptr(saved["o_s"]), _ptr(saved["o_l"]), _ptr(saved["big_l"]), _ptr(d_out), _ptr(dq),
                             _ptr(dk), _ptr(dv), _ptr(drho), _ptr(ws), n, _stream(dev))
    _raise(rc)
    return {"dq": dq, "dk": dk, "dv": dv, "drho": drho}


def soft_topk(pc, k_percent=3.0, tau=0.1):
    """soft_topk (router.hpp:126-190) on device: pc [B,H,tm,tn] fp32 -> (values [B,H,tm,tn],
    lambdas [B,H,tm]); per row the bisected shift lambda with sum_j sigma(pc/tau + lambda) = kappa.
    Raises NumericError on a row whose bisection does not converge, like the reference."""
    import torch
    if pc.dim() != 4 or pc.dtype != torch.float32 or not pc.is_contiguous():
        raise ContractError("soft_topk: contiguous fp32 scores [B, H, tm, tn]")
    B, H, tm, tn = pc.shape
    # only the score geometry is read: N = tm * tn with bq = tn, bk = tm gives tm x tn blocks
    p = FwdParams(B, H, tm * tn, 1, tn, tm, k_percent, False, False, False, True, tau)
    cp = p.c()
    values = torch.empty_like(pc)
    lambdas = torch.empty((B, H, tm), dtype=torch.float32, device=pc.device)
    _raise(lib().sla2_soft_topk(C.byref(cp), _ptr(pc), _ptr(values), _ptr(lambdas), _stream(pc.device)))
    return values, lambdas


def soft_topk_backward(values, upstream, *, tau):
    """soft_topk_backward (router.hpp:197-212) on device: the frozen-lambda gradient
    upstream * v * (1 - v) / tau of soft_topk's values [B,H,tm,tn] (fp32). tau has no default:
    it must be the tau soft_topk ran with (the reference reads it from the SoftMask)."""
    import torch
    if values.dim() != 4 or values.dtype != torch.float32 or not values.is_contiguous():
        raise ContractError("soft_topk_backward: contiguous fp32 values [B, H, tm, tn]")
    if upstream.shape != values.shape or upstream.dtype != torch.float32 or not upstream.is_contiguous():
        raise ShapeError("soft_topk_backward: shape mismatch")  # router.hpp:202-204
    B, H, tm, tn = values.shape
    p = FwdParams(B, H, tm * tn, 1, tn, tm, 100.0, False, False, False, True, tau)
    cp = p.c()
    grad = torch.empty_like(values)
    _raise(lib().sla2_soft_topk_backward(C.byref(cp), _ptr(values), _ptr(upstream), _ptr(grad), _stream(values.device)))
    return grad


def forward_soft(q, k, v, rho, values, *, bq=64, bk=64, smooth=True, saved=False):
    """sla2_forward_blockwise with Routing = SoftMask (attention.hpp:484-558), the stage-1
    training forward: fp32 q, k, v [B,H,N,d] (d, bq, bk <= 64), rho [H,tm], values [B,H,tm,tn]
    (soft_topk's). Returns out, or (out, {"o_s", "o_l", "big_l"}) with saved=True."""
    import torch
    _check_like(q, k, v)
    if q.dtype != torch.float32:
        raise ContractError("sla2_forward_soft: fp32 tensors (the stage-1 training path)")
    p = _params_from(q, bq, bk, 100.0, False, smooth, True)
    cp = p.c()
    n = int(lib().sla2_forward_soft_workspace_size(C.byref(cp)))
    if n == 0:
        _raise(lib().sla2_forward_soft(C.byref(cp), *([None] * 8), 0, None))  # raises the validation error
    dev = q.device
    if tuple(values.shape) != (p.B, p.H, p.tm, p.tn) or values.dtype != torch.float32:
        raise ShapeError("sla2_forward_blockwise: soft mask geometry mismatch")  # attention.hpp:438-440
    if tuple(rho.shape) != (p.H, p.tm):
        raise ShapeError("sla2_forward_blockwise: rho length != tm")  # attention.hpp:434
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    out = torch.empty_like(q)
    sv = None
    keep = {}
    if saved:
        keep = {"o_s": torch.empty_like(q), "o_l": torch.empty_like(q),
                "big_l": torch.empty((p.B, p.H, p.N), dtype=torch.float32, device=dev)}
        sv = _Saved(keep["o_s"].data_ptr(), keep["o_l"].data_ptr(), keep["big_l"].data_ptr(), None, None, None, None,
                    None)
    _raise(lib().sla2_forward_soft(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(rho.contiguous()),
                                   _ptr(values.contiguous()), _ptr(out), C.byref(sv) if sv is not None else None,
                                   _ptr(ws), n, _stream(dev)))
    return (out, keep) if saved else out


def sla2_attention(q, k, v, rho, proj_q, proj_k, bq=128, bk=64, k_percent=3.0, quant=False, smooth=True):
    """Tape::sla2_attention's forward (tape.hpp:263-272)."""
    return forward(q, k, v, proj_q, proj_k, rho, k_percent=k_percent, bq=bq, bk=bk, quant=quant, smooth=smooth)


def full_attention(q, k, v):
    """softmax(QK^T/sqrt d) V on the same tcgen05 kernel visiting every key block (bf16)."""
    import torch
    _check_like(q, k, v)
    p = _params_from(q, 128, 64, 100.0, False, False, True)
    cp = p.c()
    out = torch.empty_like(q)
    ws = _workspace(p, q.device)
    _raise(lib().sla2_dense_fwd(C.byref(cp), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(ws), ws.numel(),
                                _stream(q.device)))
    return out
