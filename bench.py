#!/usr/bin/env python
"""Benchmark of the BCSS sttsm hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A *step* is one full ``sttsm_bcss`` (all levels, all C blocks of the
workload) on device-resident A and X.  Default workload: BASELINE.json
``configs[1]`` (m=3, n=p=512, b_A=b_C=32, fp64).  With N>1 (launched under
torch.distributed.run, one rank per GPU) the C blocks are sharded by
top-level subtree (LPT on exact flops), A and X are broadcast once over NCCL
before timing, and no collective runs inside the timed region; the total
work is fixed, so scaling is strong.

Metric: FP64 GFLOP/s counted with the reference cost model
(bcss_costs(...).flops, costs.py:83-112) over the whole job, time = max over
ranks of the summed per-step CUDA-event times.  ``roofline`` compares the
level kernel's achieved FLOP/s with the FP64 DMMA peak measured live on this
GPU (``bcss_probe_fp64_peak``); ``e2e`` times the public host-buffer API
(pinned host A/X in, C out); ``cpu_baseline`` times the numpy oracle port on
a bounded sample of the same workload on the host cores.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port in oracle/bcss_oracle.py; the reference itself is pure Python and
cannot travel to the GPU box) on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    1: (3, 16, 16, 4, 4),
    2: (3, 512, 512, 32, 32),
    3: (4, 192, 192, 16, 16),
    4: (5, 96, 96, 8, 8),
    5: (4, 512, 256, 32, 32),
}
DEFAULT_CONFIG = 2  # BASELINE.json configs[1]
SEED = 20261019
METRIC = "sttsm FP64 GFLOP/s (blocked-alg flops)"
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x20: "sync_boost", 0x40: "sw_thermal_slowdown",
           0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget-s", type=float, default=12.0,
                    help="target CPU seconds of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                    help="S5 T(m-2) exchange: peer = the owner's kernel stores into the assignee's buffer "
                         "(CUDA IPC over NVLink), nccl = send/recv, auto = peer if every rank can map it")
    ap.add_argument("--schedule", default="auto", choices=["auto", "s1", "s5"],
                    help="multi-GPU schedule: s1 = top-level subtrees, no exchange; s5 = owners + "
                         "T(m-2) exchange + balanced subtrees (auto: s5 when s1's balance < 0.9)")
    ap.add_argument("--dense", action="store_true",
                    help="also time the dense mode-product baseline (cuBLAS) when it fits")
    ap.add_argument("--noreuse", action="store_true",
                    help="also time reuse=False (the algorithm-by-blocks without partial-symmetry reuse)")
    ap.add_argument("--e2e-sync", action="store_true",
                    help="time e2e as back-to-back synchronous calls instead of the streamed async API")
    ap.add_argument("--pipeline", type=int, default=4,
                    help="waves of the e2e transfer/compute pipeline (0 = serial copies)")
    return ap.parse_args()


def workload(cfg: int) -> dict:
    m, n, p, ba, bc = CONFIGS[cfg]
    return {"workload": f"BASELINE config {cfg}: sttsm_bcss m={m} n={n} p={p} b_A={ba} b_C={bc}",
            "m": m, "n": n, "p": p, "b_A": ba, "b_C": bc, "seed": SEED,
            "A": "random_bcss (U(-1,1) per canonical block, symmetrized diagonal blocks)",
            "X": "N(0,1) p x n"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], 0, set()
        for ln in self.lines:
            parts = [s.strip() for s in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                clk, cmax, mask = int(parts[0]), int(parts[1]), int(parts[2], 16)
            except ValueError:
                continue
            mx = max(mx, cmax)
            if mask & 0x1:  # idle sample
                continue
            sm.append(clk)
            reasons |= {name for bit, name in REASONS.items() if mask & bit}
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(a_np, x_np, m, n, p, ba, bc, budget_s: float):
    """Time the oracle port on a bounded sample of the workload: whole
    top-level subtrees (units jb_{m-1}=j), largest first, until ``budget_s``
    of CPU time is spent or the workload is complete; returns
    (GFLOP/s, description, seconds)."""
    import paper_1301_7744_b200 as bs
    from oracle import bcss_oracle as orc

    pbar = p // bc
    costs = [bs.SttsmPlan(m, n, p, ba, bc, units=[j]).stats()["flops"] for j in range(pbar)]
    done, fl = [], 0
    t0 = time.perf_counter()
    for j in sorted(range(pbar), key=lambda u: -costs[u]):
        orc.sttsm_bcss_packed(a_np, x_np, m, n, ba, bc, units=[j])
        done.append(j)
        fl += costs[j]
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    total = bs.bcss_flops(m, n, p, ba, bc)
    desc = (f"oracle port (numpy, OpenBLAS {os.cpu_count()} threads) on {len(done)} of {pbar} "
            f"top-level subtrees (jb_{m - 1} in {sorted(done)}): {fl / total:.1%} of the workload's flops")
    return fl / dt / 1e9, desc, dt


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the CPU arm runs once, on rank 0
    from oracle import bcss_oracle as orc
    import numpy as np
    import paper_1301_7744_b200 as bs

    m, n, p, ba, bc = CONFIGS[args.config]
    a_np = orc.random_bcss_packed(m, n, ba, SEED)
    x_np = np.random.default_rng(SEED + 1).standard_normal((p, n))
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(a_np, x_np, m, n, p, ba, bc, per_step / 4)
    rates, secs = [], []
    for _ in range(args.steps):
        r, desc, dt = cpu_sample(a_np, x_np, m, n, p, ba, bc, per_step)
        rates.append(r)
        secs.append(dt)
    value = sum(r * s for r, s in zip(rates, secs)) / sum(secs)
    total = bs.bcss_flops(m, n, p, ba, bc)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / (value * 1e9) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload(args.config), parallelism="cpu"),
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": os.cpu_count(),
                         "kind": "port", "sample": desc},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "ms_per_step extrapolates the sampled rate to the full workload",
    }
    print(json.dumps(line), flush=True)


def time_transfers(a_h, c_h, dev) -> dict:
    """the H2D of A and the D2H of C alone (pinned host memory,
    one copy each into/out of scratch device buffers, CUDA events), so the
    e2e number can be read against the PCIe floor."""
    import torch

    try:
        a_d = torch.empty(a_h.numel(), dtype=torch.float64, device=dev)
        c_d = torch.zeros(c_h.numel(), dtype=torch.float64, device=dev)
    except torch.cuda.OutOfMemoryError:
        torch.cuda.empty_cache()
        return {"skipped": "no free HBM for the scratch copies"}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    a_d.copy_(a_h, non_blocking=True)  # warm-up pair (first touch of the copy path)
    c_h.copy_(c_d, non_blocking=True)
    torch.cuda.synchronize()
    ev[0].record()
    a_d.copy_(a_h, non_blocking=True)
    ev[1].record()
    c_h.copy_(c_d, non_blocking=True)
    ev[2].record()
    torch.cuda.synchronize()
    h2d, d2h = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    del a_d, c_d
    torch.cuda.empty_cache()
    return {"h2d_a_ms": round(h2d, 3), "h2d_a_gbs": round(a_h.numel() * 8 / h2d / 1e6, 2),
            "d2h_c_ms": round(d2h, 3), "d2h_c_gbs": round(c_h.numel() * 8 / d2h / 1e6, 2),
            "note": "one copy each after a warm-up pair, not overlapped with anything"}


def run_dense(args, A, X, m, n, p, ba, rank, world, dev, job_ms):
    """Dense mode-product baseline (cuBLAS) on the same inputs, when it fits."""
    import torch

    from paper_1301_7744_b200 import dense as dn

    if rank != 0 or world != 1:
        return None
    need = 3 * max(n, p) ** m * 8
    free, _ = torch.cuda.mem_get_info(dev)
    if need >= 0.8 * free:
        return {"skipped": f"dense A needs ~{need / 1e9:.0f} GB"}
    a_dense = dn.bcss_to_dense_device(A, m, n, ba)
    for _ in range(2):
        dn.sttsm_dense_ttm_device(a_dense, X)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        dn.sttsm_dense_ttm_device(a_dense, X)
    s1.record()
    s1.synchronize()
    dms = s0.elapsed_time(s1) / args.steps
    dfl = dn.dense_flops(m, n, p)
    return {"ms_per_step": round(dms, 4), "flops_per_step": dfl, "tflops": round(dfl / dms / 1e9, 3),
            "speedup_bcss_vs_dense": round(dms / (job_ms / args.steps), 3),
            "impl": "dense mode-product chain, cuBLAS DGEMM via torch.tensordot"}


def run_noreuse(args, A, X, m, n, p, ba, bc, rank, world, job_ms):
    """reuse=False on the same inputs: the paper's with/without-reuse comparison."""
    import torch

    import paper_1301_7744_b200 as bs

    if rank != 0 or world != 1:
        return None
    plan = bs.SttsmPlan(m, n, p, ba, bc, reuse=False)
    C = torch.empty(plan.c_elems, dtype=torch.float64, device=A.device)
    for _ in range(2):
        plan.run(A, X, C)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        plan.run(A, X, C)
    s1.record()
    s1.synchronize()
    ms = s0.elapsed_time(s1) / args.steps
    fl = bs.bcss_flops(m, n, p, ba, bc, reuse=False)
    plan.close()
    return {"ms_per_step": round(ms, 4), "flops_per_step": fl, "tflops": round(fl / ms / 1e9, 3),
            "speedup_reuse_vs_noreuse": round(ms / (job_ms / args.steps), 3)}


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1301_7744_b200 as bs
    from paper_1301_7744_b200.distributed import S5Runner, partition_units, unit_flops
    from paper_1301_7744_b200.generate import random_bcss_device, random_matrix_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # (ranks beyond the visible GPUs wrap around: a dry run of the multi-rank
    # path on one GPU uses BCSS_BENCH_BACKEND=gloo, whose ranks never wait on
    # each other's kernels)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BCSS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    m, n, p, ba, bc = CONFIGS[args.config]
    total_flops = bs.bcss_flops(m, n, p, ba, bc)
    schedule = args.schedule
    if schedule == "auto":
        # S1 needs no exchange; take S5 only when S1's LPT balance is poor
        schedule = "s1"
        if world > 1 and m >= 3:
            costs = unit_flops(m, n, p, ba, bc)
            loads = [sum(costs[u] for u in part) for part in partition_units(costs, world)]
            if sum(costs) / world / max(loads) < 0.9:
                schedule = "s5"
    runner = None
    if schedule == "s5":
        runner = S5Runner(m, n, p, ba, bc, rank, world, dev, group=None, exchange=args.exchange)
        plans = runner.plans()
        my_flops = runner.flops
        c_elems = runner.c_elems
        plan = None
    else:
        parts = partition_units(unit_flops(m, n, p, ba, bc), world)
        plan = bs.SttsmPlan(m, n, p, ba, bc, units=parts[rank] if world > 1 else None)
        plans = [plan]
        my_flops = plan.stats()["flops"]
        c_elems = plan.c_elems
    step = runner.run if runner is not None else plan.run

    peak = bs.probe_fp64_peak()  # live FP64 DMMA peak of this GPU (roofline denominator)

    # inputs resident in HBM before timing; A and X replicated over NCCL
    if rank == 0 or world == 1:
        A = random_bcss_device(m, n, ba, SEED, device=dev)
        X = random_matrix_device(p, n, SEED + 1, device=dev)
    else:
        A = torch.empty(bs.SttsmPlan(m, n, p, ba, bc).a_elems, dtype=torch.float64, device=dev)
        X = torch.empty(p, n, dtype=torch.float64, device=dev)
    bcast_ms = None
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        dist.broadcast(A, 0)
        dist.broadcast(X, 0)
        torch.cuda.synchronize()
        bcast_ms = (time.perf_counter() - t0) * 1e3
    C = torch.zeros(c_elems, dtype=torch.float64, device=dev)
    for pl in plans:
        pl.attach_torch_workspace(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        step(A, X, C)
    torch.cuda.synchronize()
    for pl in plans:
        pl.set_timing(True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launch_ms, launch_fl = 0.0, 0
    levels: dict[int, list[float]] = {}
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            starts[i].record(stream)
            step(A, X, C)
            ends[i].record(stream)
            for pl in plans:
                for k, fl, ms in pl.launch_times():  # syncs the stream
                    launch_ms += ms
                    launch_fl += fl
                    levels.setdefault(k, [0, 0.0])
                    levels[k][0] += fl
                    levels[k][1] += ms
                launches += pl.last_launches
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    my_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    job_ms = float(t.item())
    value = total_flops * args.steps / (job_ms * 1e-3) / 1e9
    for pl in plans:
        pl.set_timing(False)

    dense_line = run_dense(args, A, X, m, n, p, ba, rank, world, dev, job_ms) if args.dense else None
    noreuse_line = run_noreuse(args, A, X, m, n, p, ba, bc, rank, world, job_ms) if args.noreuse else None
    a_np_cpu = x_np_cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        a_np_cpu, x_np_cpu = A.cpu().numpy(), X.cpu().numpy()

    # end to end through the public host-buffer API (pinned host memory)
    e2e = None
    if not args.no_e2e:
        a_h = A.cpu().pin_memory()
        x_h = X.cpu().pin_memory()
        if runner is None and world == 1 and args.pipeline:
            # the host path owns its device buffers: release the device-resident run's
            del A, X, C
            for pl in plans:
                pl.close()
            torch.cuda.empty_cache()
        c_h = torch.empty(c_elems, dtype=torch.float64).pin_memory()
        a_np, x_np, c_np = a_h.numpy(), x_h.numpy(), c_h.numpy()
        xfer = time_transfers(a_h, c_h, dev) if rank == 0 else None
        if runner is not None:
            # S5: host -> every rank's HBM, the sharded step, own C blocks back
            def e2e_step():
                A.copy_(a_h, non_blocking=True)
                X.copy_(x_h, non_blocking=True)
                step(A, X, C)
                c_h.copy_(C, non_blocking=True)
                torch.cuda.synchronize()
            plan_e2e = None
        else:
            plan_e2e = plan if (world > 1 or not args.pipeline) else bs.SttsmPlan(m, n, p, ba, bc,
                                                                                   pipeline=args.pipeline)

            def e2e_step():
                plan_e2e.run_host(a_np, x_np, c_np)
        streamed = plan_e2e is not None and plan_e2e is not plan and not args.e2e_sync
        e2e_step()  # warm: allocates device buffers
        if streamed:
            plan_e2e.run_host_async(a_np, x_np, c_np)  # warm the second buffer set
            plan_e2e.wait()
        sync_ms = None
        if streamed:
            # single-call latency of the same API, for reference
            t0 = time.perf_counter()
            for _ in range(max(1, args.steps // 2)):
                e2e_step()
            sync_ms = (time.perf_counter() - t0) / max(1, args.steps // 2) * 1e3
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if streamed:
            # K calls streamed through the asynchronous host API: every call
            # uploads its A/X and downloads its C; call i+1's upload overlaps
            # call i's compute and download (PCIe is full duplex)
            for _ in range(args.steps):
                plan_e2e.run_host_async(a_np, x_np, c_np)
            plan_e2e.wait()
        else:
            for _ in range(args.steps):
                e2e_step()
        e2e_s = time.perf_counter() - t0
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        e2e = {"value": round(total_flops * args.steps / e2e_s / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(a_h.numel() * 8 + x_h.numel() * 8),
               "d2h_bytes_per_step": int(8 * (c_h.numel() if runner is not None or world == 1 else
                                               len(plan.c_block_ranks()) * bc**m)),
               "ms_per_step": round(e2e_s / args.steps * 1e3, 3),
               "api": ("torch H2D of A/X + S5Runner.run + D2H of C, pinned host buffers" if runner is not None
                       else "SttsmPlan.run_host_async x K + wait (C ABI bcss_sttsm_run_host_async), pinned "
                            "host buffers, consecutive calls overlapped" if streamed
                       else "SttsmPlan.run_host (C ABI bcss_sttsm_run_host), pinned host buffers"),
               "sync_ms_per_call": round(sync_ms, 3) if sync_ms is not None else None,
               "pipeline_waves": args.pipeline if (plan_e2e is not None and plan_e2e is not plan) else 0,
               "transfers": xfer}
        if plan_e2e is not None and plan_e2e is not plan:
            plan_e2e.close()
        del a_h, x_h, c_h

    cpu = None
    if a_np_cpu is not None:
        rate, desc, dt = cpu_sample(a_np_cpu, x_np_cpu, m, n, p, ba, bc, args.cpu_budget_s)
        cpu = {"value": round(rate, 3), "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "port",
               "sample": desc, "seconds": round(dt, 2)}

    if rank == 0:
        achieved = launch_fl / (launch_ms * 1e-3) / 1e12
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(str(args.config))
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(job_ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(workload(args.config),
                           parallelism=(f"{schedule} x{world}" if (world > 1 or schedule == "s5") else "single"),
                           l2="flushed (256 MB write) between timed steps; A and temporaries also exceed L2"),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3),
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_source": "FP64 DMMA (mma.sync m8n8k4) probe measured live on this GPU",
                         "levels": {str(k): {"tflops": round(v[0] / (v[1] * 1e-3) / 1e12, 3),
                                             "ms_per_step": round(v[1] / args.steps, 4)}
                                    for k, v in sorted(levels.items(), reverse=True)}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "dense_baseline": dense_line,
            "noreuse_baseline": noreuse_line,
            "clocks": clocks,
            "flops_per_step": total_flops,
        }
        if bcast_ms is not None:
            line["broadcast_ms"] = round(bcast_ms, 3)
            line["rank0_flop_share"] = round(my_flops / total_flops, 4)
        if runner is not None:
            line["exchange_bytes_rank0"] = runner.exchange_bytes
            line["exchange"] = ("fused: producing kernels store into the assignee's buffer (CUDA IPC), "
                                "cross-rank order by CUDA IPC events"
                                if runner.exchange == "peer" else "NCCL send/recv")
            line["s5_helpers"] = {str(u): [h, kids] for u, (h, kids) in runner.sched["helper"].items()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
