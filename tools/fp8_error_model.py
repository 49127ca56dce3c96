"""Error model of the low-bit attention products (analysis): fp64 numpy emulation of E4M3 and
per-block INT8 rounding on random 128 x 960-key attention tiles, normwise L2 error against fp64.
Reproduces the measured FP8 P/V error (3.4-3.6e-2 on B200) and predicts the next steps (DESIGN 8)."""
import numpy as np
def e4m3(x):
    x = np.asarray(x, np.float64); s = np.sign(x); a = np.abs(x)
    a = np.minimum(a, 448.0)
    e = np.floor(np.log2(np.maximum(a, 2.0**-9)))
    e = np.maximum(e, -6)            # subnormals share the 2^-6 exponent
    q = 2.0 ** (e - 3)               # 3 mantissa bits
    return s * np.round(a / q) * q
def i8(x, s): return np.clip(np.round(x / s), -127, 127) * s
rng = np.random.default_rng(0)
n, d, nk = 128, 128, 960
errs = {k: [] for k in ("pv", "pv+qk_e4m3", "pv+qk_i8")}
for t in range(20):
    q = rng.standard_normal((n, d)); k = rng.standard_normal((nk, d)); v = rng.standard_normal((nk, d))
    def attn(q, k, pq=lambda p: p, vq=lambda v: v):
        s = q @ k.T / np.sqrt(d); m = s.max(1, keepdims=True); p = np.exp(s - m)
        return (pq(p) @ vq(v)) / p.sum(1, keepdims=True)
    ref = attn(q, k)
    vs = np.abs(v).max() / 448
    f8 = lambda: (lambda p: e4m3(p), lambda v: e4m3(v / vs) * vs)
    pq, vq = f8()
    o1 = attn(q, k, pq, vq)
    sq = np.abs(q).max() / 448; sk = np.abs(k).max() / 448
    o2 = attn(e4m3(q / sq) * sq, e4m3(k / sk) * sk, pq, vq)
    o3 = attn(i8(q, np.abs(q).max() / 127), np.concatenate([i8(k[j:j+64], np.abs(k[j:j+64]).max() / 127) for j in range(0, nk, 64)]), pq, vq)
    for key, o in (("pv", o1), ("pv+qk_e4m3", o2), ("pv+qk_i8", o3)):
        errs[key].append(np.linalg.norm(o - ref) / np.linalg.norm(ref))
for key, e in errs.items(): print(key, "L2 rel err mean %.4f" % np.mean(e))
