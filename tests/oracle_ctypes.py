"""ctypes bindings for the CPU parity oracle (TEST INFRASTRUCTURE).

Two libraries with the same entry points:
  * oracle/liboracle.so         -- the C restatement (prefix sla2o_), always built;
  * oracle/_ref/libsla2_ref.so  -- the unmodified reference headers behind extern "C"
                                   (prefix sla2r_), built only where /root/reference exists
                                   and carried to the GPU box as a prebuilt file.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libsla2_ref.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class _Opt:
    """ndpointer that also accepts None (nullable output)."""

    def __init__(self, base):
        self.base = base

    def from_param(self, obj):
        if obj is None:
            return None
        return self.base.from_param(obj)


def _build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, os.path.join(ORACLE_DIR, "liboracle.so")],
                       check=True)


class Oracle:
    """One oracle library (C port or reference) with typed numpy-facing methods."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        for s, fp, ft in (("f", _f32p, C.c_float), ("d", _f64p, C.c_double)):
            ofp = _Opt(fp)
            self._sig(f"smooth_k_{s}", [fp, _sz, _sz, fp, fp])
            self._sig(f"block_scores_{s}", [fp, fp, _sz, _sz, fp, fp, ft, _sz, _sz, fp], C.c_int)
            self._sig(f"hard_topk_{s}", [fp, _sz, _sz, C.c_double, _u8p, C.POINTER(_sz)], C.c_int)
            self._sig(f"quantize_{s}", [fp, _sz, _i8p, C.POINTER(ft)], C.c_int)
            self._sig(f"forward_blockwise_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, _u8p, fp, C.c_int,
                                                 C.c_int, fp, ofp, ofp, ofp], C.c_int)
            self._sig(f"forward_naive_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, _u8p, fp, C.c_int, fp,
                                             ofp, ofp], C.c_int)
            self._sig(f"attention_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, fp, fp, fp, C.c_double,
                                         C.c_int, C.c_int, fp, _Opt(_u8p), ofp, ofp, ofp], C.c_int)
            self._sig(f"gaussian_matrix_{s}", [fp, _sz, C.c_uint64, C.c_double], None)
            self._sig(f"random_matrix_{s}", [fp, _sz, C.c_uint64, C.c_double, C.c_double], None)
        self._sig("topk_budget", [C.c_double, _sz], _sz)
        if prefix == "sla2r_":
            for s, fp in (("f", _f32p), ("d", _f64p)):
                self._sig(f"backward_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, _u8p, fp, C.c_int, fp, fp, fp, fp, fp,
                                            fp, fp, fp], C.c_int)
                self._sig(f"soft_topk_{s}", [fp, _sz, _sz, C.c_double, C.c_float if s == "f" else C.c_double,
                                             fp, fp], C.c_int)
                self._sig(f"forward_soft_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, fp, fp, C.c_int, fp, fp, fp, fp],
                          C.c_int)
                self._sig(f"soft_topk_backward_{s}", [fp, _sz, _sz, C.c_double, C.c_float if s == "f" else C.c_double,
                                                      fp, fp], C.c_int)
                self._sig(f"forward_saved_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, _u8p, fp, C.c_int, C.c_int, fp, fp,
                                                 fp, fp, fp, fp, fp, fp], C.c_int)
                self._sig(f"block_scores_qk_{s}", [fp, fp, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int, fp], C.c_int)
                self._sig(f"rten_save_{s}", [C.c_char_p, _sz, _sz, fp], C.c_int)
                self._sig(f"rten_load_{s}", [C.c_char_p, _sz, _sz, fp], C.c_int)
        if prefix == "sla2o_":
            self._sig("set_threads", [C.c_int], None)
            for s, fp, ft in (("f", _f32p, C.c_float), ("d", _f64p, C.c_double)):
                ofp = _Opt(fp)
                # ragged extension (the C port only; the reference rejects n % block != 0)
                self._sig(f"attention_ragged_{s}", [fp, fp, fp, _sz, _sz, _sz, _sz, fp, fp, fp, C.c_double,
                                                    C.c_int, C.c_int, fp, _Opt(_u8p), ofp, ofp, ofp], C.c_int)
                self._sig(f"block_scores_ragged_{s}", [fp, fp, _sz, _sz, fp, fp, ft, _sz, _sz, fp], C.c_int)

    def _sig(self, name, argtypes, restype=C.c_int):
        fn = getattr(self.lib, self.prefix + name)
        fn.argtypes = argtypes
        fn.restype = restype
        setattr(self, "_" + name, fn)

    @staticmethod
    def _sfx(dtype):
        return "f" if np.dtype(dtype) == np.float32 else "d"

    # --- random streams of the reference's tests/test_util.hpp ---
    def gaussian(self, shape, seed, sd=1.0, dtype=np.float64):
        out = np.empty(int(np.prod(shape)), dtype=dtype)
        getattr(self, "_gaussian_matrix_" + self._sfx(dtype))(out, out.size, seed, sd)
        return out.reshape(shape)

    def uniform(self, shape, seed, lo=-1.0, hi=1.0, dtype=np.float64):
        out = np.empty(int(np.prod(shape)), dtype=dtype)
        getattr(self, "_random_matrix_" + self._sfx(dtype))(out, out.size, seed, lo, hi)
        return out.reshape(shape)

    def topk_budget(self, k_percent, tn):
        return int(self._topk_budget(k_percent, tn))

    def smooth_k(self, k):
        n, d = k.shape
        kt = np.empty_like(k)
        mu = np.empty(d, dtype=k.dtype)
        getattr(self, "_smooth_k_" + self._sfx(k.dtype))(np.ascontiguousarray(k), n, d, kt, mu)
        return kt, mu

    def block_scores(self, q, k, proj_q, proj_k, bq, bk, tau=0.1):
        n, d = q.shape
        dt = q.dtype
        pc = np.empty((n // bq if bq else 0, n // bk if bk else 0), dtype=dt)
        rc = getattr(self, "_block_scores_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), n, d,
            np.ascontiguousarray(proj_q, dtype=dt), np.ascontiguousarray(proj_k, dtype=dt),
            tau, bq, bk, pc)
        _check(rc)
        return pc

    def hard_topk(self, pc, k_percent):
        tm, tn = pc.shape
        mask = np.empty((tm, tn), dtype=np.uint8)
        kappa = _sz(0)
        rc = getattr(self, "_hard_topk_" + self._sfx(pc.dtype))(
            np.ascontiguousarray(pc), tm, tn, k_percent, mask, C.byref(kappa))
        _check(rc)
        return mask, int(kappa.value)

    def quantize(self, x):
        x = np.ascontiguousarray(x)
        codes = np.empty(x.shape, dtype=np.int8)
        scale = (C.c_float if x.dtype == np.float32 else C.c_double)(0)
        getattr(self, "_quantize_" + self._sfx(x.dtype))(x.ravel(), x.size, codes.ravel(),
                                                         C.byref(scale))
        return codes, scale.value

    def forward_blockwise(self, q, k, v, bq, bk, mask, rho, quant=False, smooth=True):
        n, d = q.shape
        dt = q.dtype
        out = np.empty((n, d), dt)
        o_s = np.empty((n, d), dt)
        o_l = np.empty((n, d), dt)
        big_l = np.empty(n, dt)
        rc = getattr(self, "_forward_blockwise_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(mask, dtype=np.uint8), np.ascontiguousarray(rho, dtype=dt),
            int(quant), int(smooth), out, o_s, o_l, big_l)
        _check(rc)
        return out, o_s, o_l, big_l

    def forward_saved(self, q, k, v, bq, bk, mask, rho, quant=False, smooth=True):
        """sla2_forward_blockwise with the whole SLA2ForwardSaved (reference only): dict of out,
        o_s, o_l, big_l, h_blocks [tm,d,d], z_blocks [tm,d], q_phi, k_phi."""
        n, d = q.shape
        dt = q.dtype
        tm = n // bq
        r = {"out": np.empty((n, d), dt), "o_s": np.empty((n, d), dt), "o_l": np.empty((n, d), dt),
             "big_l": np.empty(n, dt), "h_blocks": np.empty((tm, d, d), dt), "z_blocks": np.empty((tm, d), dt),
             "q_phi": np.empty((n, d), dt), "k_phi": np.empty((n, d), dt)}
        rc = getattr(self, "_forward_saved_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(mask, dtype=np.uint8), np.ascontiguousarray(rho, dtype=dt), int(quant), int(smooth),
            r["out"], r["o_s"], r["o_l"], r["big_l"], r["h_blocks"], r["z_blocks"], r["q_phi"], r["k_phi"])
        _check(rc)
        return r

    def block_scores_qk(self, q, k, qi0, bq, kj0, bk, quant=False):
        """detail::block_scores_qk (attention.hpp:372-394) of one block pair (reference only); k is
        the (smoothed) K~ the forward passes."""
        n, d = q.shape
        s = np.empty((bq, bk), q.dtype)
        rc = getattr(self, "_block_scores_qk_" + self._sfx(q.dtype))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), n, d, qi0, bq, kj0, bk, int(quant), s)
        _check(rc)
        return s

    def forward_naive(self, q, k, v, bq, bk, mask, rho, smooth=True):
        n, d = q.shape
        dt = q.dtype
        out = np.empty((n, d), dt)
        o_s = np.empty((n, d), dt)
        o_l = np.empty((n, d), dt)
        rc = getattr(self, "_forward_naive_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(mask, dtype=np.uint8), np.ascontiguousarray(rho, dtype=dt),
            int(smooth), out, o_s, o_l)
        _check(rc)
        return out, o_s, o_l

    def attention(self, q, k, v, bq, bk, proj_q, proj_k, rho, k_percent, quant=False, smooth=True):
        """Tape::sla2_attention forward composition (tape.hpp:263-272) for one (b, h)."""
        n, d = q.shape
        dt = q.dtype
        out = np.empty((n, d), dt)
        o_s = np.empty((n, d), dt)
        o_l = np.empty((n, d), dt)
        big_l = np.empty(n, dt)
        mask = np.empty((n // bq, n // bk), np.uint8)
        rc = getattr(self, "_attention_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(proj_q, dtype=dt), np.ascontiguousarray(proj_k, dtype=dt),
            np.ascontiguousarray(rho, dtype=dt), k_percent, int(quant), int(smooth), out, mask,
            o_s, o_l, big_l)
        _check(rc)
        return out, mask, o_s, o_l, big_l


    def block_scores_ragged(self, q, k, proj_q, proj_k, bq, bk, tau=0.1):
        """Ragged extension of block_scores (C port only): partial last blocks pooled over their
        own rows."""
        n, d = q.shape
        dt = q.dtype
        pc = np.empty((-(-n // bq), -(-n // bk)), dtype=dt)
        rc = getattr(self, "_block_scores_ragged_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), n, d,
            np.ascontiguousarray(proj_q, dtype=dt), np.ascontiguousarray(proj_k, dtype=dt),
            tau, bq, bk, pc)
        _check(rc)
        return pc

    def attention_ragged(self, q, k, v, bq, bk, proj_q, proj_k, rho, k_percent, quant=False, smooth=True):
        """Ragged extension of attention(): n need not be divisible by bq / bk (C port only)."""
        n, d = q.shape
        dt = q.dtype
        tm, tn = -(-n // bq), -(-n // bk)
        out = np.empty((n, d), dt)
        o_s = np.empty((n, d), dt)
        o_l = np.empty((n, d), dt)
        big_l = np.empty(n, dt)
        mask = np.empty((tm, tn), np.uint8)
        rc = getattr(self, "_attention_ragged_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(proj_q, dtype=dt), np.ascontiguousarray(proj_k, dtype=dt),
            np.ascontiguousarray(rho, dtype=dt), k_percent, int(quant), int(smooth), out, mask,
            o_s, o_l, big_l)
        _check(rc)
        return out, mask, o_s, o_l, big_l


    def backward(self, q, k, v, bq, bk, mask, rho, d_out, smooth=True):
        """sla2_backward (attention.hpp:610-809) on the reference's own forward state, hard mask
        (reference library only). Returns dq, dk, dv, drho, o_s, o_l, big_l."""
        n, d = q.shape
        dt = q.dtype
        outs = [np.empty((n, d), dt) for _ in range(3)] + [np.empty(n // bq, dt)] + \
            [np.empty((n, d), dt) for _ in range(2)] + [np.empty(n, dt)]
        rc = getattr(self, "_backward_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(mask, dtype=np.uint8), np.ascontiguousarray(rho, dtype=dt), int(smooth),
            np.ascontiguousarray(d_out, dtype=dt), *outs)
        _check(rc)
        return tuple(outs)

    def soft_topk(self, pc, k_percent, tau):
        """soft_topk (router.hpp:126-190), reference library only. Returns (values, lambdas)."""
        tm, tn = pc.shape
        values = np.empty((tm, tn), pc.dtype)
        lambdas = np.empty(tm, pc.dtype)
        _check(getattr(self, "_soft_topk_" + self._sfx(pc.dtype))(np.ascontiguousarray(pc), tm, tn, k_percent, tau,
                                                                  values, lambdas))
        return values, lambdas

    def soft_topk_backward(self, pc, k_percent, tau, upstream):
        """soft_topk_backward (router.hpp:197-212) on soft_topk(pc)'s mask, reference library only."""
        tm, tn = pc.shape
        grad = np.empty((tm, tn), pc.dtype)
        _check(getattr(self, "_soft_topk_backward_" + self._sfx(pc.dtype))(
            np.ascontiguousarray(pc), tm, tn, k_percent, tau, np.ascontiguousarray(upstream, dtype=pc.dtype), grad))
        return grad

    def forward_soft(self, q, k, v, bq, bk, values, rho, smooth=True):
        """sla2_forward_blockwise with a SoftMask (attention.hpp:484-558), reference library only.
        Returns out, o_s, o_l, big_l."""
        n, d = q.shape
        dt = q.dtype
        outs = [np.empty((n, d), dt) for _ in range(3)] + [np.empty(n, dt)]
        _check(getattr(self, "_forward_soft_" + self._sfx(dt))(
            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v), n, d, bq, bk,
            np.ascontiguousarray(values, dtype=dt), np.ascontiguousarray(rho, dtype=dt), int(smooth), *outs))
        return tuple(outs)

    # --- RTEN1 through the reference's sla2::rten (tensor_io.hpp), reference library only ---
    def rten_save(self, path, a):
        a = np.ascontiguousarray(a)
        rows, cols = (a.shape if a.ndim == 2 else (0, a.shape[0]))
        _check(getattr(self, "_rten_save_" + self._sfx(a.dtype))(str(path).encode(), rows, cols, a))

    def rten_load(self, path, shape, dtype=np.float32):
        out = np.empty(shape, dtype)
        rows, cols = (shape if len(shape) == 2 else (0, shape[0]))
        _check(getattr(self, "_rten_load_" + self._sfx(dtype))(str(path).encode(), rows, cols, out))
        return out


class OracleError(Exception):
    pass


class ShapeError(OracleError):
    pass


class NumericError(OracleError):
    pass


def _check(rc):
    if rc == 0:
        return
    if rc == 1:
        raise ShapeError("shape_error")
    if rc == 2:
        raise NumericError("numeric_error")
    raise OracleError(f"oracle error {rc}")


_port = None
_ref = None


def port() -> Oracle:
    """The C restatement (always available; built on demand with gcc)."""
    global _port
    if _port is None:
        _build_oracle()
        _port = Oracle(ORACLE_SO, "sla2o_")
    return _port


def ref():
    """The unmodified reference behind extern "C", or None when it was not built here."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Oracle(REF_SO, "sla2r_")
    return _ref
