"""The exact (reference-rounding) kernels must not contain fused packed multiply-adds.

ptxas contracts a packed FMUL2 that feeds a packed FADD2 into one FFMA2 (a single rounding),
even when both come from `__fmul2_rn` / `__fadd2_rn` or explicit `.rn` PTX. The router's score
and projection chains (matrix.hpp:101-135, router.hpp:87-102) and the QAT O fold
(attention.hpp:516-529) round the product and the sum separately, so their kernels keep the
sums scalar. This test reads the built library's SASS (CPU only: cuobjdump cross-reads sm_100a).
"""
import os
import re
import shutil
import subprocess
from functools import lru_cache

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2602_12675_b200", "libsla2_b200.so")

# kernels whose float arithmetic is bit-exact with the reference's two-rounding chains
EXACT = ("router_rows_kernel", "project_kernel", "pool_project_kernel", "colmean", "kprep_kernel",
         "router_scores_topk_kernel")


@lru_cache(maxsize=1)
def _functions():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    if not os.path.exists(LIB):
        pytest.skip("libsla2_b200.so not built")
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name:
            funcs[name].append(line)
    return funcs


def test_exact_chains_have_no_ffma2():
    funcs = _functions()
    checked = 0
    for name, body in funcs.items():
        if not any(k in name for k in EXACT):
            continue
        checked += 1
        bad = [ln.strip() for ln in body if re.search(r"\bFFMA2\b", ln)]
        assert not bad, f"{name}: fused packed multiply-add in an exact chain: {bad[:3]}"
    assert checked >= 6, f"expected the router kernels in the library, found {checked}"


def test_qat_fold_has_no_ffma2_beyond_the_exponent():
    # attn_i8: the only FFMA2 is the exponent argument S * log2e - m (a tolerance-level step, as in
    # the reference's expf); the fold O = fl(fl(O corr) + fl(acc sP sV)) must stay unfused
    funcs = _functions()
    name = next((n for n in funcs if "sla2_attn_i8_kernel" in n), None)
    if name is None:
        pytest.skip("attn_i8 kernel not in this build")
    n = sum(1 for ln in funcs[name] if re.search(r"\bFFMA2\b", ln))
    assert n <= 32, f"{n} FFMA2 in {name}: the O fold was contracted"
