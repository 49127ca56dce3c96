#!/usr/bin/env python
"""SLA2 forward benchmark (BASELINE.json metric) on 1..8 B200s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1|cfg2|cfg2pad|cfg3|cfg3fp8|cfg4|cfg4fp8|cfg5|cfg5fp8]
                  [--impl b200|reference] [--scaling weak|strong]

A step is one full SLA2 forward (router + linear precompute + sparse/linear/blend kernel) over
one synthetic batch of the workload, inputs resident in HBM. value = effective attention
TFLOPS = 4 N^2 d B H / t of the whole job (all ranks' heads / max rank time).

Multi-GPU: `--gpus N` re-launches itself under torch.distributed.run when WORLD_SIZE is unset
(one process per GPU, NCCL; gloo and a CPU stand-in when no CUDA device exists -- a plumbing
check that reports no value). With N > 1 the default is STRONG scaling of BASELINE configs[3]
(cfg4: 40 heads sharded 20/10/5 per rank, no collective in the data path); at N = 1 it is
configs[1] (cfg2). After the timed region rank 0 all-gathers every head's mask and two sampled
output heads and checks them against the oracle (the `parity` block, untimed).

--config cfg5 runs the BASELINE configs[4] sweep (sparsity x N vs the dense kernel of the same
build) and prints one JSON line with every point.

--impl reference times the reference's own CPU implementation (oracle/_ref/libsla2_ref.so
built from the unmodified headers; the oracle port when absent) on the host cores, one head of
the same workload per step, rank 0 only.

bench.py executes oracle/ only in untimed legs: the CPU baseline / reference arm, and the
parity block (the checker). The timed product path is the CUDA library alone.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SLA2 attn fwd ms & effective TFLOPS at Wan2.1 shape, 97% sparsity, 1-8 GPU"
CONFIGS = {
    # configs[1]: the true Wan2.1-1.3B attention shape, N = 32760 (ragged: the last query block
    # has 120 rows and the last key block 56 keys; tests/test_ragged.py)
    "cfg2": dict(workload="wan2.1-1.3B-480p attention (BASELINE configs[1])", B=1, H=12, N=32760, d=128, bq=128,
                 bk=64, k_percent=3.0, bf16=True, quant=False),
    # the same padded to the block multiple (the reference's own shape rule), for comparison
    "cfg2pad": dict(workload="wan2.1-1.3B-480p attention, N padded to 32768", B=1, H=12, N=32768, d=128, bq=128,
                    bk=64, k_percent=3.0, bf16=True, quant=False),
    # the INT8 QAT path keeps the reference's divisibility rule (N padded to 32768)
    "cfg3": dict(workload="wan2.1-1.3B-480p attention, INT8 QAT (BASELINE configs[2])", B=1, H=12, N=32768,
                 d=128, bq=128, bk=64, k_percent=3.0, bf16=True, quant=True),
    # configs[2]'s low-bit P/V product (FP8 PV): E4M3 P, V and phi(K~) on kind::f8f6f4, bf16 Q K^T,
    # at the true N = 32760; not a reference mode (the reference is INT8-only), so the oracle is the
    # unquantized reference; the output bar is the FP8 one (1e-1 max normwise, tests/test_gpu_fp8.py)
    "cfg3fp8": dict(workload="wan2.1-1.3B-480p attention, FP8 P/V low-bit mode (BASELINE configs[2])", B=1, H=12,
                    N=32760, d=128, bq=128, bk=64, k_percent=3.0, bf16=True, quant="fp8"),
    "cfg4fp8": dict(workload="wan2.1-14B-720p attention, FP8 P/V low-bit mode", B=1, H=40, N=75600, d=128,
                    bq=128, bk=64, k_percent=3.0, bf16=True, quant="fp8"),
    "cfg4": dict(workload="wan2.1-14B-720p attention (BASELINE configs[3])", B=1, H=40, N=75600, d=128, bq=128,
                 bk=64, k_percent=3.0, bf16=True, quant=False),
    "cfg1": dict(workload="fp32 CPU-oracle case (BASELINE configs[0])", B=1, H=2, N=4096, d=64, bq=64, bk=64,
                 k_percent=10.0, bf16=False, quant=False),
    # configs[4]: the sweep (H = 12, the 1.3B model's heads); see sweep()
    "cfg5fp8": dict(workload="the configs[4] sweep in the FP8 P/V low-bit mode", B=1, H=12, N=32768, d=128, bq=128,
                    bk=64, k_percent=3.0, bf16=True, quant="fp8"),
    "cfg5": dict(workload="sparsity {80,85,90,95,97}% x N {8K..128K} vs dense (BASELINE configs[4])", B=1, H=12,
                 N=32768, d=128, bq=128, bk=64, k_percent=3.0, bf16=True, quant=False),
}
SWEEP_SPARSITY = (80, 85, 90, 95, 97)
SWEEP_N = (8192, 16384, 32768, 65536, 131072)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sustained": p.get("bf16_tflops_sustained"),
                "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


def eff_flops(c):
    # the paper's effective FLOPs, 4 N^2 d per head = flops_full (accounting.hpp:39-45)
    from paper_2602_12675_b200.accounting import GeometryConfig, flops_full
    return flops_full(GeometryConfig(c["N"], c["d"], c["B"] * c["H"], 1, 1))


def flops_model(c, kappa, tn, ms):
    """The reference's analytic SLA2 cost at the kept fraction (flops_sla2, accounting.hpp:47-77)."""
    from paper_2602_12675_b200.accounting import GeometryConfig, flops_sla2
    r = flops_sla2(GeometryConfig(c["N"], c["d"], c["B"] * c["H"], 1, 1), 1.0 - kappa / tn, c["bq"], c["bk"])
    return {"source": "flops_sla2 (accounting.hpp:47-77) at sparsity 1 - kappa / tn", "full": r.full,
            "sparse_branch": r.sparse_branch, "linear_branch": r.linear_branch, "router": r.router,
            "total": r.total, "savings": r.savings, "tflops_on_model_total": r.total / (ms * 1e-3) / 1e12}


def geometry(c):
    tm, tn = -(-c["N"] // c["bq"]), -(-c["N"] // c["bk"])  # ceil: ragged N has a partial last block
    kappa = max(1, min(tn, int(round(c["k_percent"] / 100.0 * tn))))
    return tm, tn, kappa


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while running."""

    def __init__(self, dev_index):
        self.samples = []
        self.proc = None
        self.dev = dev_index
        self.t_on = None

    def start(self):
        try:
            import torch
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.dev).uuid)
        except Exception:
            uuid = str(self.dev)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", uuid, f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def mark_on(self):
        self.t_on = time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [p for (t, p) in self.samples if self.t_on is None or t >= self.t_on]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][1]),
                "power_w_max": max((num(r[2]) or 0.0) for r in rows), "samples": len(rows), "reasons": reasons}


# ------------------------------------------------------------------------------ CPU reference
def cpu_reference_run(c, steps, warmup, threads=None):
    """Times the reference CPU path (Tape::sla2_attention forward composition per head) on
    host cores. Returns (per-step seconds list, kind, cores, N timed)."""
    threads = threads or os.cpu_count() or 1
    os.environ["SLA2_THREADS"] = str(threads)  # read once by max_worker_threads (common.hpp:31-43)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ctypes as oc
    from sla2_testlib import make_inputs
    o = oc.ref()
    kind = "reference"
    if o is None:
        o = oc.port()
        o._set_threads(threads)
        kind = "port"
    # the reference rejects N % block != 0 (attention.hpp:39-41): a ragged N is timed at the next
    # multiple of the blocks (0.02% more work at 32760 -> 32768)
    blk = max(c["bq"], c["bk"])
    n_ref = -(-c["N"] // blk) * blk
    q, k, v, pq, pk, rho = make_inputs(1, 1, n_ref, c["d"], seed=7, bf16=c["bf16"], bq=c["bq"], bk=c["bk"])
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        o.attention(q[0, 0], k[0, 0], v[0, 0], c["bq"], c["bk"], pq[0], pk[0], rho[0], c["k_percent"],
                    quant=c["quant"] is True)
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    return times, kind, threads, n_ref


# ------------------------------------------------------------------------------ launching
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(n):
    """`python bench.py --gpus N` outside torchrun: one process per GPU under
    torch.distributed.run (the driver's own launch line), rendezvous on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def time_events(fn, reps, flush=None):
    """Median ms of fn() over reps CUDA-event timed calls (L2 flushed before each)."""
    import torch
    dts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        dts.append(e0.elapsed_time(e1))
    return statistics.median(dts)


# ------------------------------------------------------------------------------ parity (untimed)
def parity_block(c, masks_all, outs, dev, seed_base, dtype):
    """Rank 0: the gathered masks of every head and the sampled output heads vs the oracle on
    the same inputs, regenerated from the per-head seeds (dist.head_inputs)."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ctypes as oc
    from paper_2602_12675_b200 import dist as sd
    from sla2_testlib import verify_gathered
    threads = os.cpu_count() or 1
    os.environ.setdefault("SLA2_THREADS", str(threads))
    oc.port()._set_threads(threads)
    tm = geometry(c)[0]

    def regen(h):
        q, k, v, pq, pk, rho = sd.head_inputs(h, c["N"], c["d"], tm, dtype, dev, seed_base)
        return tuple(x.float().cpu().numpy() for x in (q, k, v, pq, pk, rho))

    t0 = time.perf_counter()
    res = verify_gathered(masks_all.cpu().numpy(), {h: o.float().cpu().numpy() for h, o in outs.items()}, regen,
                          c["k_percent"], c["bq"], c["bk"], quant=c["quant"] is True,
                          tol=0.1 if c["quant"] == "fp8" else 1e-2)  # FP8 bar: tests/test_gpu_fp8.py
    res["check_s"] = round(time.perf_counter() - t0, 2)
    return res


# ------------------------------------------------------------------------------ cfg5 sweep
def sweep(args, dev, name="cfg5"):
    """BASELINE configs[4]: SLA2 forward (graph replay) vs the dense tcgen05 kernel of the same
    build and cuDNN SDPA, over sparsity x N, H = 12, bf16."""
    import torch
    import torch.nn.functional as F
    import paper_2602_12675_b200 as sla2
    from paper_2602_12675_b200 import dist as sd
    base = CONFIGS[name]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    points = []
    for N in SWEEP_N:
        c = dict(base, N=N)
        tm = geometry(c)[0]
        q, k, v, pq, pk, rho = sd.shard_inputs(0, c["H"], 1, N, c["d"], tm, torch.bfloat16, dev)
        flops = eff_flops(c)
        dense_ms = time_events(lambda: sla2.full_attention(q, k, v), 3, flush)
        sdpa_ms = time_events(lambda: F.scaled_dot_product_attention(q, k, v), 3, flush)
        for sp in SWEEP_SPARSITY:
            kp = 100.0 - sp
            kw = dict(k_percent=kp, bq=c["bq"], bk=c["bk"], quant=c["quant"])
            g = sla2.CapturedForward(q, k, v, pq, pk, rho, **kw)
            for _ in range(max(args.warmup, 3)):
                g()
            ms = time_events(g, max(args.steps, 5), flush)
            kappa = geometry(dict(c, k_percent=kp))[2]
            points.append({"N": N, "sparsity_pct": sp, "kappa": kappa, "tn": geometry(c)[1], "sla2_ms": ms,
                           "sla2_tflops": flops / (ms * 1e-3) / 1e12, "dense_ms": dense_ms,
                           "speedup_vs_dense": dense_ms / ms, "sdpa_ms": sdpa_ms, "speedup_vs_sdpa": sdpa_ms / ms})
            del g
        del q, k, v
        torch.cuda.empty_cache()
    return points


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: cfg2 on 1 GPU, cfg4 (heads sharded) on more")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="weak: each rank runs the full workload; strong: heads sharded over ranks "
                         "(default: strong when N > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg_name = args.config or ("cfg2" if world == 1 else "cfg4")
    scaling = args.scaling or ("weak" if world == 1 else "strong")
    c = dict(CONFIGS[cfg_name])
    tm, tn, kappa = geometry(c)
    cfg_out = {"workload": c["workload"], "name": cfg_name, "B": c["B"], "H": c["H"], "N": c["N"], "d": c["d"],
               "bq": c["bq"], "bk": c["bk"], "k_percent": c["k_percent"], "kappa": kappa, "sparsity": 1 - kappa / tn,
               "quant": {True: "int8", False: "none"}.get(c["quant"], c["quant"]),
               "parallelism": (f"heads-replicated x{world} (weak)" if scaling == "weak"
                               else f"heads sharded over {world} ranks (strong)")}

    if args.impl == "reference":
        if rank != 0:
            return
        times, kind, cores, n_ref = cpu_reference_run(c, args.steps, args.warmup)
        t = statistics.median(times)
        val = 4.0 * n_ref ** 2 * c["d"] / t / 1e12
        sample = (f"1 of {c['B'] * c['H']} (b,h) heads per step: smooth_k + block_scores + hard_topk + "
                  f"sla2_forward_blockwise<float>, SLA2_THREADS={cores}"
                  + (f", N={n_ref} (the reference rejects N={c['N']})" if n_ref != c["N"] else ""))
        line = {"metric": METRIC, "value": val, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg_out, "impl": "reference",
                "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": cores, "kind": kind, "sample": sample},
                "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "full_forward_ms_extrapolated": t * 1e3 * c["B"] * c["H"]}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2602_12675_b200 import dist as sd

    has_cuda = torch.cuda.is_available()
    if not has_cuda:
        return standin_main(args, c, cfg_out, world, rank, scaling)
    import paper_2602_12675_b200 as sla2
    import ctypes as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if cfg_name in ("cfg5", "cfg5fp8"):
        if rank == 0:
            pts = sweep(args, dev, cfg_name)
            at = next(p for p in pts if p["N"] == 32768 and p["sparsity_pct"] == 97)
            print(json.dumps({"metric": METRIC, "value": at["sla2_tflops"], "unit": "TFLOPS", "n_gpus": 1,
                              "steps": args.steps, "warmup": args.warmup, "ms_per_step": at["sla2_ms"],
                              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
                              "data": "synthetic", "config": dict(cfg_out, value_at="97%, N=32768"),
                              "sweep": pts}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return
    sampler = ClockSampler(local)
    sampler.start()

    # synthetic inputs per GLOBAL head (dist.head_inputs): weak scaling gives every rank the
    # whole workload under its own seed range; strong scaling shards the heads contiguously
    B, H_total, N, d = c["B"], c["H"], c["N"], c["d"]
    h0, h1 = sd.head_range(H_total, world, rank) if scaling == "strong" else (0, H_total)
    H = h1 - h0
    seed_base = 1234 + (rank * 1000003 if scaling == "weak" else 0)
    dt = torch.bfloat16 if c["bf16"] else torch.float32
    q, k, v, pq, pk, rho = sd.shard_inputs(h0, h1, B, N, d, tm, dt, dev, seed_base)
    out = torch.empty_like(q)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    kw = dict(k_percent=c["k_percent"], bq=c["bq"], bk=c["bk"], quant=c["quant"], out=out)

    def eager_step():
        sla2.forward(q, k, v, pq, pk, rho, **kw)

    for _ in range(args.warmup):
        eager_step()
    torch.cuda.synchronize()
    launches_per_step = sla2.last_launch_count()
    # the timed steps replay the forward captured once as a CUDA graph (same kernels, same
    # inputs and output; the host launch work is gone)
    graph = sla2.CapturedForward(q, k, v, pq, pk, rho, **kw)

    def step():
        graph()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # stage timing pass (dominant-kernel roofline), untimed for value
    sla2.enable_stage_timing(True)
    stages = []
    for _ in range(min(args.steps, 20)):
        flush.zero_()
        eager_step()
        stages.append(sla2.last_stage_ms(timeline=True))
    sla2.enable_stage_timing(False)
    st_med = [statistics.median(s[i] for s in stages) for i in range(len(stages[0]))]
    timeline = dict(zip(("mu_ready", "query_side_done", "key_prep_done", "router_back_done", "linear_prep_done"),
                        st_med[4:9]))

    # clock pre-roll (~1 s of back-to-back steps), then the timed region
    t_end = time.time() + 1.0
    sampler.mark_on()
    while time.time() < t_end:
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    wall0 = time.perf_counter()
    for s in range(args.steps):
        flush.zero_()
        ev0[s].record()
        step()
        ev1[s].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    sampler.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    t_max = sd.max_over_ranks(total_ms, device=dev)  # the job is as slow as its slowest rank
    ms_per_step = t_max / args.steps
    job_flops = eff_flops(c) * (world if scaling == "weak" else 1)
    value = job_flops / (ms_per_step * 1e-3) / 1e12
    flops = eff_flops(dict(c, H=H))  # this rank's share, for the per-kernel roofline below
    clocks = sampler.summary()

    # verification (untimed): every head's mask and two sampled output heads reach rank 0 over
    # NCCL (strong: the sharded job's heads; weak: rank 0's own workload)
    parity = None
    if not args.no_parity and B == 1:
        _, mask_local = sla2.forward(q, k, v, pq, pk, rho, k_percent=c["k_percent"], bq=c["bq"], bk=c["bk"],
                                     quant=c["quant"], return_mask=True)
        out_local = sla2.forward(q, k, v, pq, pk, rho, **kw)
        if scaling == "strong":
            masks_all = sd.gather_head_shards(mask_local[0], H_total, world, rank)
            outs = sd.gather_sampled_heads(out_local[0], [0, H_total - 1], H_total, world, rank)
        else:
            masks_all, outs = mask_local[0], {0: out_local[0, 0], H_total - 1: out_local[0, H_total - 1]}
        if rank == 0:
            parity = parity_block(c, masks_all, outs, dev, seed_base, dt)
        del mask_local, out_local

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk_ = peaks()
    # dominant kernel = the fused sparse + linear + blend kernel (stage 2): 4 N kappa bk d flops
    # of QK^T and PV over the kept blocks plus 2 N d^2 of phi(Q) Hc, per (b, h)
    sparse_alg = B * H * (4.0 * N * kappa * c["bk"] * d + 2.0 * N * d * d)
    sparse_ms = st_med[2]
    achieved = sparse_alg / (sparse_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(cfg_name, {}).get("sparse_kernel_dram_bytes_per_launch")
    except Exception:
        pass
    if c["quant"] == "fp8":
        # PV and phi(K~)^T V on kind::f8f6f4 (twice the bf16 rate), Q K^T and the phi(Q) Hc product
        # on kind::f16: the bf16 peak is the conservative denominator
        kern, peak, peak_src = ("sla2_sparse_v2_kernel<F8> (E4M3 P / V / phi(K~))", pk_["bf16"],
                                pk_["src"] + " burst bf16 (MEASURED_PEAKS.json)")
    elif c["quant"]:
        # the QAT stage: K~ codes (quant_prep_kernel), the bf16 linear branch (sla2_linsel_kernel)
        # and the INT8 softmax branch (sla2_attn_i8_kernel: QK^T and PV on tcgen05 kind::i8, K = 32
        # per instruction at the kind::f16 issue rate, tools/mb_umma.cu -> twice the bf16 peak)
        kern = "quant_prep_kernel (K~ codes) + sla2_linsel_kernel + sla2_attn_i8_kernel"
        peak, peak_src = 2 * pk_["bf16"], pk_["src"] + " bf16 burst x 2 (kind::i8)"
    elif c["bf16"]:
        kern, peak, peak_src = "sla2_sparse_v2_kernel", pk_["bf16"], pk_["src"] + " burst bf16 (MEASURED_PEAKS.json)"
    else:
        kern, peak, peak_src = "sla2_sparse_f32_kernel", pk_["bf16"], pk_["src"] + " burst bf16 (MEASURED_PEAKS.json)"
    roofline = {"bound": "tensor", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "peak_src": peak_src,
                "algorithmic_flops_per_launch": sparse_alg, "launch_ms": sparse_ms,
                "traffic_src": "profiles/ncu_summary.json (ncu --set full dram__bytes_read+write, per launch)"}

    extra = {}
    # dense tcgen05 attention of the same build (the north-star's 15x comparison) and cuDNN SDPA
    if not args.no_dense and c["bf16"]:
        for _ in range(2):
            sla2.full_attention(q, k, v)
        torch.cuda.synchronize()
        dense_ms = time_events(lambda: sla2.full_attention(q, k, v), 3, flush)
        extra["dense_same_build"] = {"ms": dense_ms, "tflops": flops / (dense_ms * 1e-3) / 1e12,
                                     "speedup_sla2_vs_dense": dense_ms / ms_per_step,
                                     "dense_frac_of_peak": flops / (dense_ms * 1e-3) / 1e12 / pk_["bf16"]}
        try:
            import torch.nn.functional as F
            for _ in range(2):
                F.scaled_dot_product_attention(q, k, v)
            torch.cuda.synchronize()
            sdpa_ms = time_events(lambda: F.scaled_dot_product_attention(q, k, v), 3, flush)
            extra["torch_sdpa_ms"] = sdpa_ms
            extra["speedup_vs_sdpa"] = sdpa_ms / ms_per_step
        except Exception as ex:  # context only
            extra["torch_sdpa_ms"] = f"unavailable: {ex}"

    # end to end through the C ABI with host buffers (sla2_forward_host), copies inside
    e2e = None
    if not args.no_e2e:
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        hpq, hpk, hrho = (x.cpu().pin_memory() for x in (pq, pk, rho))
        hout = torch.empty_like(hq).pin_memory()
        cp = sla2.FwdParams(B, H, N, d, c["bq"], c["bk"], c["k_percent"], c["bf16"], c["quant"]).c()
        L = sla2.lib()

        def host_step():
            rc = L.sla2_forward_host(C.byref(cp), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), hpq.data_ptr(),
                                     hpk.data_ptr(), hrho.data_ptr(), hout.data_ptr(), None)
            if rc != 0:
                raise RuntimeError(L.sla2_last_error().decode())
        for _ in range(2):
            host_step()
        n_e2e = max(3, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            host_step()
        e2e_s = (time.perf_counter() - t0) / n_e2e
        esz = 2 if c["bf16"] else 4
        e2e = {"value": flops / e2e_s / 1e12, "unit": "TFLOPS", "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": 3 * B * H * N * d * esz + 2 * H * d * d * 4 + H * tm * 4,
               "d2h_bytes_per_step": B * H * N * d * esz, "api": "sla2_forward_host (C ABI, pinned host buffers)",
               "ranks": f"rank 0's shard ({H} heads)" if world > 1 else "whole workload"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        times, kind, cores, n_ref = cpu_reference_run(c, 1, 0)
        t = statistics.median(times)
        cpu = {"value": 4.0 * n_ref ** 2 * d / t / 1e12, "unit": "TFLOPS", "cores": cores, "kind": kind,
               "sample": f"1 of {B * H} heads ({t:.2f} s): Tape::sla2_attention forward composition, "
                         f"SLA2_THREADS={cores}" + (f", N={n_ref} (the reference rejects N={N})" if n_ref != N else ""),
               "ms_per_head": t * 1e3,
               "full_forward_ms_extrapolated": t * 1e3 * B * H}

    line = {"metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16" if c["bf16"] else "f32",
            "data": "synthetic (torch.randn N(0,1) per head seed, proj = I + 0.05 N(0,1), rho ~ U(-1,1))",
            "config": dict(cfg_out, l2="flushed between timed steps (256 MiB write, outside the events)",
                           launch="one CUDA-graph replay of the captured forward per step"),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
            "stages_ms": {"router": st_med[0], "linear_prep": st_med[1], "sparse_kernel": sparse_ms,
                          "total": st_med[3]},
            "timeline_ms": timeline, "flops_model": flops_model(c, kappa, tn, ms_per_step),
            "wall_s_timed_region": wall, **extra}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def standin_main(args, c, cfg_out, world, rank, scaling):
    """No CUDA device: the multi-rank plumbing alone over gloo (shard planning, barriers,
    max-over-ranks, the mask / sampled-output gathers and the rank-0 verify), with each rank's
    shard computed by the CPU oracle as a STAND-IN. No product code runs, so no value is
    reported; this is what `python bench.py --gpus 2` checks on a CPU box."""
    import torch
    import torch.distributed as dist
    from paper_2602_12675_b200 import dist as sd
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from sla2_testlib import oracle_attention_any
    if world > 1:
        dist.init_process_group("gloo")
    # a small shape of the same workload family: the oracle runs the stand-in compute
    c = dict(c, N=min(c["N"], 2048 if c["N"] % 64 == 0 else 2000), H=min(c["H"], 4 * world), B=1)
    tm, tn, kappa = geometry(c)
    cfg_out = dict(cfg_out, N=c["N"], H=c["H"], kappa=kappa, sparsity=1 - kappa / tn)
    H_total = c["H"]
    h0, h1 = sd.head_range(H_total, world, rank)
    dev = torch.device("cpu")
    dt = torch.bfloat16 if c["bf16"] else torch.float32
    t0 = time.perf_counter()
    masks, outs = [], []
    for h in range(h0, h1):
        q, k, v, pq, pk, rho = (x.float().numpy() for x in sd.head_inputs(h, c["N"], c["d"], tm, dt, dev))
        o, m = oracle_attention_any(q, k, v, pq, pk, rho, c["bq"], c["bk"], c["k_percent"], quant=c["quant"] is True)[:2]
        masks.append(torch.from_numpy(m))
        outs.append(torch.from_numpy(o))
    t_max = sd.max_over_ranks((time.perf_counter() - t0) * 1e3)
    masks_all = sd.gather_head_shards(torch.stack(masks), H_total, world, rank)
    sampled = sd.gather_sampled_heads(torch.stack(outs), [0, H_total - 1], H_total, world, rank)
    if rank == 0:
        parity = parity_block(c, masks_all, sampled, dev, 1234, dt)
        print(json.dumps({"metric": METRIC, "value": None, "unit": "TFLOPS", "n_gpus": world, "steps": 0,
                          "warmup": 0, "ms_per_step": None, "higher_is_better": True, "scaling": scaling,
                          "vs_baseline": None, "dtype": "bf16" if c["bf16"] else "f32", "data": "synthetic",
                          "config": dict(cfg_out, parallelism=f"heads sharded over {world} ranks"),
                          "standin": "no CUDA device: CPU oracle stand-in compute over gloo (plumbing check, "
                                     "no product code, no value)",
                          "standin_compute_ms_max_over_ranks": t_max, "parity": parity}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
