#!/usr/bin/env python
"""SLA2 forward benchmark (BASELINE.json metric) on 1..8 B200s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|cfg3|cfg4|cfg1] [--impl b200|reference]

A step is one full SLA2 forward (router + linear precompute + sparse/linear/blend kernel) over
one synthetic batch of the workload, inputs resident in HBM. value = effective attention
TFLOPS = 4 N^2 d B H / t, whole job (sum over ranks / max rank time). Multi-GPU
is weak scaling: every rank runs its own full workload (heads are independent, no collective
in the data path); NCCL all-gathers a per-rank output checksum afterwards for verification
only (untimed). L2 is flushed (256 MiB write) between timed steps, outside the events.

--impl reference times the reference's own CPU implementation (oracle/_ref/libsla2_ref.so
built from the unmodified headers; the oracle port when absent) on the host cores, one head of
the same workload per step, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
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
    "cfg4": dict(workload="wan2.1-14B-720p attention (BASELINE configs[3])", B=1, H=40, N=75600, d=128, bq=128,
                 bk=64, k_percent=3.0, bf16=True, quant=False),
    "cfg1": dict(workload="fp32 CPU-oracle case (BASELINE configs[0])", B=1, H=2, N=4096, d=64, bq=64, bk=64,
                 k_percent=10.0, bf16=False, quant=False),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sustained": p.get("bf16_tflops_sustained"),
                "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


def eff_flops(c):
    return 4.0 * c["N"] ** 2 * c["d"] * c["B"] * c["H"]


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
    host cores. Returns (per-step seconds list, kind, cores)."""
    import numpy as np
    threads = threads or os.cpu_count() or 1
    os.environ["SLA2_THREADS"] = str(threads)  # read once by max_worker_threads (common.hpp:31-43)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_ctypes as oc
    from sla2_testlib import make_inputs
    o = oc.ref()
    kind = "reference"
    if o is None:
        o = oc.port()
        o.set_threads(threads) if hasattr(o, "set_threads") else o._set_threads(threads)
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
                    quant=c["quant"])
        dt = time.perf_counter() - t0
        if s >= warmup:
            times.append(dt)
    return times, kind, threads, n_ref


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank runs the full workload; strong: heads sharded over ranks")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = dict(CONFIGS[args.config])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    tm, tn = -(-c["N"] // c["bq"]), -(-c["N"] // c["bk"])  # ceil: ragged N has a partial last block
    kappa = max(1, min(tn, round(c["k_percent"] / 100.0 * tn)))
    cfg_out = {"workload": c["workload"], "B": c["B"], "H": c["H"], "N": c["N"], "d": c["d"], "bq": c["bq"],
               "bk": c["bk"], "k_percent": c["k_percent"], "kappa": kappa, "sparsity": 1 - kappa / tn,
               "quant": "int8" if c["quant"] else "none",
               "parallelism": (f"heads-replicated x{world} (weak)" if args.scaling == "weak"
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
                "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg_out, "impl": "reference",
                "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": cores, "kind": kind, "sample": sample},
                "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "full_forward_ms_extrapolated": t * 1e3 * c["B"] * c["H"]}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2602_12675_b200 as sla2
    from paper_2602_12675_b200 import dist as sd
    import ctypes as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    sampler = ClockSampler(local)
    sampler.start()

    # synthetic inputs, per-rank seed. weak: every rank runs the full workload (its own batch);
    # strong: the workload's heads are sharded over the ranks (contiguous, no data exchange)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    B, H_total, N, d = c["B"], c["H"], c["N"], c["d"]
    h0, h1 = sd.head_range(H_total, world, rank) if args.scaling == "strong" else (0, H_total)
    H = h1 - h0
    dt = torch.bfloat16 if c["bf16"] else torch.float32
    q = torch.randn((B, H, N, d), generator=g, device=dev).to(dt)
    k = torch.randn((B, H, N, d), generator=g, device=dev).to(dt)
    v = torch.randn((B, H, N, d), generator=g, device=dev).to(dt)
    eye = torch.eye(d, device=dev)[None]
    pq = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    pk = (eye + 0.05 * torch.randn((H, d, d), generator=g, device=dev)).contiguous()
    rho = (torch.rand((H, tm), generator=g, device=dev) * 2 - 1).contiguous()
    out = torch.empty_like(q)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    kw = dict(k_percent=c["k_percent"], bq=c["bq"], bk=c["bk"], quant=c["quant"], out=out)
    if os.environ.get("SLA2_BENCH_INEXACT_MU"):  # experiment only: tree-reduced mean (mask may differ)
        kw["exact_mu"] = False

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
    # verification only (untimed): all-gather per-rank output checksums over NCCL
    finite = all(x == x and abs(x) != float("inf") for x in sd.gather_checksums(out.float(), device=dev))
    ms_per_step = t_max / args.steps
    flops = eff_flops(c)  # whole-workload flops of one rank's job (weak) / of the sharded job (strong)
    value = (world if args.scaling == "weak" else 1) * flops / (ms_per_step * 1e-3) / 1e12
    flops = eff_flops(dict(c, H=H))  # this rank's share, for the per-kernel roofline below
    clocks = sampler.summary()

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk_ = peaks()
    # dominant kernel = the fused sparse + linear + blend kernel (stage 2)
    sparse_alg = B * H * (4.0 * N * kappa * c["bk"] * d + 2.0 * N * d * d)
    sparse_ms = st_med[2]
    achieved = sparse_alg / (sparse_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get(args.config, {}).get("sparse_kernel_dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": "sla2_sparse_bf16_kernel" if c["bf16"] else "sla2_sparse_f32_kernel",
                "achieved": achieved, "peak": pk_["bf16"], "unit": "TFLOP/s", "frac": achieved / pk_["bf16"],
                "traffic": traffic, "peak_src": pk_["src"] + " burst bf16 (MEASURED_PEAKS.json)",
                "algorithmic_flops_per_launch": sparse_alg, "launch_ms": sparse_ms}

    extra = {}
    # dense tcgen05 attention of the same build (the north-star's 15x comparison)
    if not args.no_dense and c["bf16"]:
        for _ in range(2):
            sla2.full_attention(q, k, v)
        torch.cuda.synchronize()
        dts = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sla2.full_attention(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            dts.append(e0.elapsed_time(e1))
        dense_ms = statistics.median(dts)
        extra["dense_same_build"] = {"ms": dense_ms, "tflops": flops / (dense_ms * 1e-3) / 1e12,
                                     "speedup_sla2_vs_dense": dense_ms / ms_per_step,
                                     "dense_frac_of_peak": flops / (dense_ms * 1e-3) / 1e12 / pk_["bf16"]}
        try:
            import torch.nn.functional as F
            for _ in range(2):
                F.scaled_dot_product_attention(q, k, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            F.scaled_dot_product_attention(q, k, v)
            e1.record()
            torch.cuda.synchronize()
            extra["torch_sdpa_ms"] = e0.elapsed_time(e1)
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
               "d2h_bytes_per_step": B * H * N * d * esz, "api": "sla2_forward_host (C ABI, pinned host buffers)"}

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
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16" if c["bf16"] else "f32",
            "data": "synthetic (torch.randn N(0,1), proj = I + 0.05 N(0,1), rho ~ U(-1,1))",
            "config": dict(cfg_out, l2="flushed between timed steps (256 MiB write, outside the events)",
                           launch="one CUDA-graph replay of the captured forward per step"),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
            "stages_ms": {"router": st_med[0], "linear_prep": st_med[1], "sparse_kernel": sparse_ms,
                          "total": st_med[3]},
            "timeline_ms": timeline,
            "wall_s_timed_region": wall, "output_finite": finite, **extra}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
