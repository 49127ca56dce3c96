"""Shared helpers for the parity tests: seeded synthetic inputs in the bench's layout and
per-(b, h) oracle evaluation (TEST INFRASTRUCTURE)."""
from __future__ import annotations

import numpy as np

import oracle_ctypes as oc


def make_inputs(B, H, N, d, seed=0, sigma=1.0, bf16=True, k_percent=3.0, bq=128, bk=64):
    """Q, K, V ~ N(0, sigma^2) (rounded to bf16 when bf16), proj = I + 0.05 N(0,1) per head
    (test_gradients.cpp:143-148), rho ~ U(-1, 1) per head and query block (:149).
    Returns numpy float32 arrays holding exactly the values the GPU receives."""
    rng = np.random.default_rng(seed)
    q = (rng.standard_normal((B, H, N, d)) * sigma).astype(np.float32)
    k = (rng.standard_normal((B, H, N, d)) * sigma).astype(np.float32)
    v = rng.standard_normal((B, H, N, d)).astype(np.float32)
    if bf16:
        q, k, v = (bf16_round(x) for x in (q, k, v))
    pq = (np.eye(d, dtype=np.float32)[None] + 0.05 * rng.standard_normal((H, d, d))).astype(np.float32)
    pk = (np.eye(d, dtype=np.float32)[None] + 0.05 * rng.standard_normal((H, d, d))).astype(np.float32)
    rho = rng.uniform(-1, 1, (H, N // bq)).astype(np.float32)
    return q, k, v, pq, pk, rho


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 -> float32 (what torch .to(bfloat16) does)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def to_dev(x, dtype, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to(device=device).to(dtype)


def oracle_head(q, k, v, pq, pk, rho, bq, bk, k_percent, quant=False, smooth=True, which="port"):
    """Tape::sla2_attention forward for one (b, h) slice on the CPU oracle (float)."""
    o = oc.port() if which == "port" else oc.ref()
    return o.attention(q, k, v, bq, bk, pq, pk, rho, k_percent, quant=quant, smooth=smooth)


def oracle_router_head(q, k, pq, pk, bq, bk, k_percent, smooth=True, which="port"):
    o = oc.port() if which == "port" else oc.ref()
    kt = o.smooth_k(k)[0] if smooth else k
    pc = o.block_scores(q, kt, pq, pk, bq, bk)
    mask, kappa = o.hard_topk(pc, k_percent)
    return pc, mask, kappa


def oracle_router_any(q, k, pq, pk, bq, bk, k_percent, smooth=True):
    """Router for one (b, h) at any N: the unmodified reference (oracle/_ref) when N divides into
    blocks and it was built here, else the C port's ragged extension (pinned to the reference on
    divisible N, tests/test_ragged.py). Returns (pc, mask, kappa, which)."""
    n = q.shape[0]
    r = oc.ref()
    if n % bq == 0 and n % bk == 0 and r is not None:
        kt = r.smooth_k(k)[0] if smooth else k
        pc = r.block_scores(q, kt, pq, pk, bq, bk)
        mask, kappa = r.hard_topk(pc, k_percent)
        return pc, mask, kappa, "reference"
    o = oc.port()
    kt = o.smooth_k(k)[0] if smooth else k
    pc = o.block_scores_ragged(q, kt, pq, pk, bq, bk) if (n % bq or n % bk) else o.block_scores(q, kt, pq, pk, bq, bk)
    mask, kappa = o.hard_topk(pc, k_percent)
    return pc, mask, kappa, "port"


def oracle_attention_any(q, k, v, pq, pk, rho, bq, bk, k_percent, quant=False):
    """Tape::sla2_attention forward for one (b, h) at any N: the reference when N divides (and it
    was built here), else the port's ragged extension. Returns (out, mask, o_s, o_l, L, which)."""
    n = q.shape[0]
    r = oc.ref()
    if n % bq == 0 and n % bk == 0 and r is not None:
        return (*r.attention(q, k, v, bq, bk, pq, pk, rho, k_percent, quant=quant), "reference")
    return (*oc.port().attention_ragged(q, k, v, bq, bk, pq, pk, rho, k_percent, quant=quant), "port")


def mask_to_idx(mask):
    return [np.nonzero(row)[0].astype(np.int32) for row in mask]


def rel_err(got, ref):
    """Normwise relative errors: (max|d| / max|ref|, ||d||_2 / ||ref||_2)."""
    d = np.asarray(got, np.float64) - np.asarray(ref, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.abs(d).max() / max(np.abs(r).max(), 1e-30)), float(np.linalg.norm(d) / max(np.linalg.norm(r), 1e-30))
