"""Host mirror of the reference's metric accounting (accounting.hpp:10-77): the analytic FLOPs of
full attention and of the SLA2 blockwise kernel per geometry. bench.py's effective TFLOPS use
flops_full (4 N^2 d per head); flops_sla2 gives the algorithmic split reported next
to it. Same names, fields, arithmetic order (float64) and errors (ShapeError) as the reference."""
from __future__ import annotations

from dataclasses import dataclass

from . import ShapeError


@dataclass
class GeometryConfig:
    """accounting.hpp:10-26: tokens, head dim, heads, layers, denoising steps."""
    n: int = 0
    d: int = 0
    heads: int = 1
    layers: int = 1
    steps: int = 1

    def validate(self) -> None:
        if self.n == 0 or self.d == 0 or self.heads == 0 or self.layers == 0 or self.steps == 0:
            raise ShapeError("GeometryConfig: all fields must be positive")

    def multiplier(self) -> float:
        return float(self.heads) * float(self.layers) * float(self.steps)


@dataclass
class FlopsReport:
    """accounting.hpp:28-37."""
    full: float = 0.0
    sparse_branch: float = 0.0
    linear_branch: float = 0.0
    router: float = 0.0
    total: float = 0.0
    sparsity: float = 0.0
    savings: float = 0.0            # 1 - total / full
    overhead_fraction: float = 0.0  # (linear + router) / full, independent of sparsity


def flops_full(g: GeometryConfig) -> float:
    """Full attention: 4 N^2 d per head per layer per step (accounting.hpp:39-45)."""
    g.validate()
    n, d = float(g.n), float(g.d)
    return 4.0 * n * n * d * g.multiplier()


def flops_sla2(g: GeometryConfig, sparsity: float, bq: int, bk: int) -> FlopsReport:
    """The blockwise kernel's analytic cost (accounting.hpp:47-77): the kept fraction of the full
    QK^T + PV work, the linear branch's accumulator form, the router's pooled projections and
    compressed score matmul (block counts as real ratios)."""
    g.validate()
    if not (sparsity >= 0.0 and sparsity < 1.0):
        raise ShapeError("flops_sla2: sparsity must be in [0, 1)")
    n, d = float(g.n), float(g.d)
    tmr, tnr = n / float(bq), n / float(bk)
    mult = g.multiplier()
    r = FlopsReport()
    r.sparsity = sparsity
    r.full = flops_full(g)
    r.sparse_branch = (1.0 - sparsity) * 4.0 * n * n * d * mult
    r.linear_branch = (4.0 * n * d * d + 2.0 * n * d) * mult
    r.router = (2.0 * tmr * tnr * d + 2.0 * tmr * d * d + 2.0 * tnr * d * d + 2.0 * n * d) * mult
    r.total = r.sparse_branch + r.linear_branch + r.router
    r.savings = 1.0 - r.total / r.full
    r.overhead_fraction = (r.linear_branch + r.router) / r.full
    return r
