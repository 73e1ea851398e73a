#!/usr/bin/env python
"""bench.py -- Crius hot path on B200: full-space Cell estimation + one round.

One "step" = one pass of the whole hot path over the synthetic
workload with profiles resident in HBM: enumerate every Cell (K1), estimate
every Cell (fused DP + plan cost + argmin), all-gather the per-Cell records
(N > 1, NCCL), and one scheduling round (K5/K6) with decisions read back.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl crius|reference]

Default workload: BASELINE.json configs[3] (the north_star target: 10k-job
Philly-like trace, 4 GPU types x 512 = 2048 GPUs, stages 1-16, DP x TP <= 64).
Prints ONE JSON line on rank 0.  `value` = Cell-plan evaluations per second of
the whole step (sum of plans of all Cells / step time), aggregated over all
ranks (strong scaling: the Cell space is fixed and sharded).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2403_16125_b200 import workload as W  # noqa: E402

ALU_OPS_PER_DP_PROBE = 8      # one binary-search probe of the stage DP
ALU_OPS_PER_STAGE_EVAL = 40   # one (plan, stage) cost evaluation
SM_COUNT = 148
# int32 lanes per SM that execute the estimator's integer work: the ALU and the
# FMA pipes of the 4 SMSPs, 16 lanes each (4 x (16 + 16) = 128)
INT_LANES_PER_SM = 128
# k_round (one 256-thread CTA, sequential by definition) has no throughput
# roofline; its structural floor is its chain of CTA-wide barriers (counted by
# the kernel: every Phase A iteration, every sequence recomputation, every
# ScaleResource evaluation, every Phase B batch) x the measured __syncthreads
# latency at 256 threads on this B200: 29.1 cycles
# (profiles/r2/latency_microbench.txt).
BARRIER_CYCLES = 29.1
ROUND_THREADS = 256


def round_floor(st, sm_mhz):
    n = st["cta_barriers"]
    return n, n * BARRIER_CYCLES / (sm_mhz * 1e3)  # barriers, ms


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="crius", choices=["crius", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--variant", default=None)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4,
                    help="N=1 e2e: crius_update_estimate with the row upload pipelined in this "
                         "many job ranges (0: update + enumerate + estimate, unpipelined)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--assembly", type=int, default=0,
                    help="NEXT-1: 1 = per-stage DP-only/TP-only (paper), 2 = every factorisation")
    ap.add_argument("--form", type=int, default=1, help="pipeline form for --assembly (1 = paper)")
    ap.add_argument("--tune", action="store_true",
                    help="NEXT-3: after --assembly 1, tune every Cell in its favoured halves")
    ap.add_argument("--paper-stages", action="store_true",
                    help="NEXT-2: the paper's stage determination instead of the min-max DP")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1 exchange: NCCL all-gather + compaction (north_star), or the fused "
                         "exchange (estimate kernel stores into every rank's window over NVLink)")
    return ap.parse_args()


def workload_name(a):
    v = f"-{a.variant}" if a.variant else ""
    s = f"x{a.scale}" if a.scale != 1 else ""
    m = f"-assembly{a.assembly}form{a.form}" if getattr(a, "assembly", 0) else ""
    m += "-tuned" if getattr(a, "tune", False) else ""
    m += "-paperstages" if getattr(a, "paper_stages", False) else ""
    return f"cfg{a.config}{v}{s}{m}"


def config_dict(a, pr, n_cells, n_plans, world, flush):
    return {"workload": workload_name(a), "jobs": pr.n_jobs, "gpu_types": pr.n_types,
            "cluster_gpus": int(pr.cap.sum()), "cells": int(n_cells), "cell_plans": int(n_plans),
            "gpu_set": ["paper3", "all_pow2"][pr.gpu_set], "s_max": pr.s_max, "g_max": pr.g_max,
            "microbatches": "4S" if pr.b_mode == 0 else [int(b) for b in pr.b_values],
            "search_depth": pr.depth,
            "parallelism": f"cell-range sharding x{world} + " + (
                "fused P2P exchange (estimate kernel -> NVLink peer windows)"
                if world > 1 and getattr(a, "gather", "nccl") == "p2p" else "all-gather"),
            "l2": "flushed between steps (256 MiB write)" if flush else "not flushed",
            "activation_model": "stage-input activations per sample (DESIGN R-1: 2*s*h per "
                                "transformer block, GPipe re-materialisation), not SURVEY "
                                "§8(d)'s 34*s*h + 5*heads*s^2; it decides which plans pass the "
                                "memory filter (PAPER.md:390)"}


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region through NVML
    (every 2 ms); falls back to nvidia-smi if NVML is unavailable."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception:
            self.nv = None

    def run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                if nv is not None:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    names = [n for n, attr in self.REASONS if r & getattr(nv, attr, 0)]
                    self.rows.append((float(sm), float(self.smax), names))
                else:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip().split(",")
                    self.rows.append((float(out[0]), float(out[1]), []))
            except Exception:
                pass
            self.stop.wait(0.002 if nv is not None else 0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for r in self.rows for n in r[2]})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


# --------------------------------------------------------------- helpers
def algorithmic_ops(pr, cells, units):
    """DP probes S_top*L*ceil(log2 L) per unit + stage evaluations
    sum(nplans * S) per Cell, for the Cells of the given unit set."""
    job, S, npl = cells["job"], cells["S"], cells["nplans"]
    stage_evals = int((npl.astype(np.int64) * S).sum())
    unit = job.astype(np.int64) * pr.n_types + cells["type"]
    stop = np.zeros(units, np.int64)
    np.maximum.at(stop, unit, S)
    L = np.repeat(pr.n_layers.astype(np.int64), pr.n_types)
    lg = np.maximum(1, np.ceil(np.log2(np.maximum(L, 2)))).astype(np.int64)
    probes = int((stop * L * lg).sum())
    return probes, stage_evals, ALU_OPS_PER_DP_PROBE * probes + ALU_OPS_PER_STAGE_EVAL * stage_evals


def algorithmic_bytes(pr, cells):
    """SURVEY §8(d) algorithmic HBM bytes of one full estimate: per unit (job,
    type) the compute planes k <= log2(max g) it needs (int32 per layer; the
    kernel stages exactly these), per job its per-layer rows once (w, act, bnd,
    tpv int64 + tpn int32 = 36 B per layer; the other types' units re-read them
    from L2), per Cell its table entry (G, S int32 + plan offset int64) read and
    its 16-byte record written."""
    T, K1e = pr.n_types, pr.k_max + 1
    ng = pr.ng.astype(np.int64)
    L = pr.n_layers.astype(np.int64)
    planes = 0
    for t in range(T):
        cap = int(pr.cap[t])
        if pr.gpu_set == 1:
            gtop = np.full_like(ng, cap)
        else:
            gtop = np.where(2 * ng <= cap, 2 * ng, np.where(ng <= cap, ng, ng // 2))
        g = np.minimum(np.maximum(gtop, 1), pr.g_max)
        k1 = np.minimum(np.floor(np.log2(g)).astype(np.int64) + 1, K1e)
        planes += int((k1 * L * 4).sum())
    n_cells = len(cells["job"])
    return planes + int(L.sum()) * 36 + n_cells * (16 + 16)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def committed_traffic(name):
    p = os.path.join(ROOT, "profiles", "estimate_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        e = d.get(name)
        return None if e is None else e["bytes_per_launch"]
    return None


# --------------------------------------------------------------- reference arm (oracle)
def run_reference(a, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build()
    pr = W.make_config(a.config, variant=a.variant, scale=a.scale)
    o = oracle.Oracle(pr)
    cells = o.enumerate()
    n, p = o.count()
    # bounded sample: whole-space estimate of the first units covering <= ~2.5 s of CPU work
    c1 = len(cells["job"])
    t0 = time.perf_counter()
    o.estimate(cells, 0, min(c1, 2000))
    per_cell = (time.perf_counter() - t0) / min(c1, 2000)
    c1 = int(min(c1, max(2000, 2.5 / max(per_cell, 1e-9))))
    sample_plans = int(cells["nplans"][:c1].sum())
    full = c1 == len(cells["job"])
    times = []
    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        t_ns, _ = o.estimate(cells, 0, c1)
        if full:
            o.round(cells, t_ns)
        dt = time.perf_counter() - t0
        if i >= a.warmup:
            times.append(dt)
    tot = sum(times)
    value = sample_plans * a.steps / tot
    sample = (f"full workload ({n} Cells, {p} plans) estimate + round" if full else
              f"first {c1} of {n} Cells ({sample_plans} plans), estimate only")
    line = {"metric": "Cell-plan evaluations/sec", "value": value, "unit": "cell-plans/s",
            "impl": "reference", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded)",
            "config": config_dict(a, pr, n, p, world, False),
            "cpu_baseline": {"value": value, "unit": "cell-plans/s", "cores": 1, "kind": "oracle",
                             "sample": sample, "cpu_model": host_cpu()},
            "e2e": {"value": value, "unit": "cell-plans/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_PAR = {}


def _par_estimate(rng):
    import oracle
    o = oracle.Oracle(_PAR["pr"])
    o.estimate(_PAR["cells"], rng[0], rng[1])
    return rng[1] - rng[0]


def cpu_parallel(pr, cells, c1):
    """the oracle's estimation of Cells [0, c1) sharded over P =
    (usable host cores) forked processes by contiguous work-balanced Cell ranges
    (weight nplans * S); the round stays single-threaded."""
    import multiprocessing as mp
    P = max(1, len(os.sched_getaffinity(0)))
    w = (cells["nplans"][:c1].astype(np.int64) * cells["S"][:c1]).cumsum()
    cuts = [0] + [int(np.searchsorted(w, w[-1] * r / P)) for r in range(1, P)] + [c1]
    ranges = [(cuts[r], cuts[r + 1]) for r in range(P) if cuts[r + 1] > cuts[r]]
    _PAR.update(pr=pr, cells=cells)
    ctx = mp.get_context("fork")
    with ctx.Pool(P) as pool:
        pool.map(_par_estimate, [(0, 1)] * P)  # fork + oracle load outside the timed region
        t0 = time.perf_counter()
        pool.map(_par_estimate, ranges, chunksize=1)
        dt = time.perf_counter() - t0
    plans = int(cells["nplans"][:c1].sum())
    return {"value": plans / dt, "unit": "cell-plans/s", "cores": P, "estimate_s": dt,
            "sample": f"estimate of Cells [0, {c1}) on {len(ranges)} processes, no round"}


def host_cpu():
    """The host CPU model name (report it beside the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(a, pr):
    """The oracle as it stands on this host, one core, bounded sample (~10-30 s);
    plus its estimation sharded over every host core."""
    out = _cpu_baseline(a, pr)
    out["cpu_model"] = host_cpu()
    out["host_threads"] = os.cpu_count()
    return out


def _cpu_baseline(a, pr):
    import oracle
    oracle.build()
    o = oracle.Oracle(pr)
    cells = o.enumerate()
    n = len(cells["job"])
    t0 = time.perf_counter()
    c1 = min(n, 2000)
    o.estimate(cells, 0, c1)
    dt = time.perf_counter() - t0
    budget = 12.0
    if n > c1 and dt * n / c1 > budget:  # estimate a prefix of the Cell space only
        c1 = int(min(n, max(c1, budget * c1 / max(dt, 1e-9))))
        t0 = time.perf_counter()
        o.estimate(cells, 0, c1)
        dt = time.perf_counter() - t0
        plans = int(cells["nplans"][:c1].sum())
        return {"value": plans / dt, "unit": "cell-plans/s", "cores": 1, "kind": "oracle",
                "sample": f"estimate of the first {c1} of {n} Cells ({plans} plans), no round",
                "parallel": cpu_parallel(pr, cells, c1)}
    t0 = time.perf_counter()
    t_ns, _ = o.estimate(cells)
    t1 = time.perf_counter()
    o.round(cells, t_ns)
    t2 = time.perf_counter()
    plans = int(cells["nplans"].sum())
    par = cpu_parallel(pr, cells, n)
    par["value"] = plans / (par["estimate_s"] + (t2 - t1))
    par["sample"] = (f"full workload: estimate on {par['cores']} processes "
                     f"{par['estimate_s']:.3f} s + single-threaded round {t2 - t1:.2f} s")
    return {"value": plans / (t2 - t0), "unit": "cell-plans/s", "cores": 1, "kind": "oracle",
            "sample": f"full workload: estimate {t1 - t0:.2f} s + round {t2 - t1:.2f} s",
            "estimate_s": t1 - t0, "round_s": t2 - t1, "parallel": par}


# --------------------------------------------------------------- our arm
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2403_16125_b200 as pkg
    from paper_2403_16125_b200 import sharded

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    pr = W.make_config(a.config, variant=a.variant, scale=a.scale)
    cr = pkg.Crius(pr, device=local)
    n_cells, n_plans, n_units = cr.enumerate()
    plan = sharded.ShardPlan(cr, world)
    ub = plan.unit_begin
    mine = cr.new_results(plan.chunk)
    gathered = cr.new_results(world * plan.chunk) if world > 1 else None
    full = cr.new_results(n_cells) if world > 1 else None
    cells_h = {k: v.cpu().numpy() for k, v in cr.cells().items()}
    stage_tp = (torch.empty((max(n_cells, 1), cr.max_stages()), dtype=torch.int8, device=dev)
                if a.assembly else None)
    xch = None
    if world > 1 and a.gather == "p2p":
        if a.paper_stages or a.assembly:
            raise SystemExit("--gather p2p: the fused exchange covers the D1 estimator only")
        xch = sharded.PeerExchange(cr, rank, world)
    flush = not a.no_flush
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(times=None):
        e0, e1, e2, e3, e4 = ev(), ev(), ev(), ev(), ev()
        e0.record(stream)
        cr.enumerate()
        if world > 1:
            sharded.ShardPlan(cr, world)  # partition is part of the step (a tiny kernel + D2H)
        e1.record(stream)
        if a.paper_stages:
            cr.estimate_paper_stages(int(ub[rank]), int(ub[rank + 1]), out=mine)
        elif a.assembly:
            cr.estimate_assembled(a.assembly, a.form, int(ub[rank]), int(ub[rank + 1]), out=mine,
                                  stage_tp=stage_tp)
            if a.tune:
                cr.tune_assembled(stage_tp, a.form, int(ub[rank]), int(ub[rank + 1]), out=mine)
        elif xch is not None:
            cr.estimate_exchange(int(ub[rank]), int(ub[rank + 1]))
        else:
            cr.estimate(int(ub[rank]), int(ub[rank + 1]), out=mine)
        e2.record(stream)
        if xch is not None:
            res = cr.exchange_wait()
        elif world > 1:
            dist.all_gather_into_tensor(gathered, mine[:plan.chunk])
            res = cr.compact(gathered, plan.chunk, world, plan.cell_begin, out=full)
        else:
            res = mine
        e3.record(stream)
        dec = cr.schedule_round(res)
        e4.record(stream)
        if times is not None:
            times.append((e0, e1, e2, e3, e4))
        return dec

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = cr.launches()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(a.steps):
            if flush:
                flush_buf.fill_(1)
            step(times)
        torch.cuda.synchronize()
    launches = cr.launches() - launches0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    seg = np.array([[t[i].elapsed_time(t[i + 1]) for i in range(4)] for t in times])  # ms
    step_ms = seg.sum(axis=1)
    tot_ms = float(step_ms.sum())
    tot_t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot_t, op=dist.ReduceOp.MAX)
    tot_ms = float(tot_t.item())
    ms_per_step = tot_ms / a.steps
    value = n_plans * a.steps / (tot_ms / 1e3)
    est_ms = float(np.median(seg[:, 1]))

    # estimate-kernel roofline (ALU-bound; HBM fraction reported beside it)
    probes, stage_evals, ops = algorithmic_ops(pr, cells_h, n_units)
    r_units = int(ub[rank + 1] - ub[rank])
    frac_units = r_units / max(n_units, 1)
    peaks, src = load_peaks()
    clocks = clk.summary()
    peak_ops = SM_COUNT * INT_LANES_PER_SM * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    achieved_ops = ops * frac_units / (est_ms / 1e3)
    alg_bytes = algorithmic_bytes(pr, cells_h) * frac_units
    hbm = alg_bytes / (est_ms / 1e3) / 1e9

    # e2e through the public API: pinned host inputs -> update (H2D) -> enumerate
    # -> estimate -> round (decisions D2H), same metric
    e2e = None
    if not a.no_e2e:
        pin = {}
        for k in ("c", "w", "act", "bnd", "tpv", "tpn", "job_id", "submit", "ng", "gb", "kst",
                  "n_layers", "layer_off", "cap", "gpn", "mem", "alpha_in", "beta_in", "alpha_x",
                  "beta_x"):
            arr = np.ascontiguousarray(getattr(pr, k))
            tt = torch.from_numpy(arr).pin_memory()
            pin[k] = tt
            setattr(pr, k, tt.numpy())
        # a rank uploads the per-job arrays and the per-layer rows of its own jobs
        # (SURVEY §8(e)); the partition depends on the per-job arrays only, which
        # do not change between steps here, so the setup plan's job range holds
        j0, j1 = plan.job_range(rank, pr.n_types) if world > 1 else (0, pr.n_jobs)
        row_keys = ("c", "w", "act", "bnd", "tpv", "tpn")
        l0, l1 = int(pr.layer_off[j0]), int(pr.layer_off[j1])
        h2d = sum(int(t.numel() * t.element_size()) for k, t in pin.items() if k not in row_keys)
        h2d += sum(int(pin[k].element_size()) * (int(pin[k].numel()) // pr.total_layers) * (l1 - l0)
                   for k in row_keys)
        d2h = pr.n_jobs * 8 + pr.n_types * 4 + 8 + 3 * 8 + (pr.n_jobs + 1) * 4

        def e2e_step():
            # the user's call sequence: new profiles from host memory -> decisions on host
            if world > 1:
                cr.update(pr, j0, j1)
                cr.enumerate()
                pl = sharded.ShardPlan(cr, world)
                assert pl.job_range(rank, pr.n_types) == (j0, j1)
                res = (xch.estimate_all(pl) if xch is not None else
                       sharded.estimate_all(cr, pl, rank, mine=mine, gathered=gathered, full=full))
            elif a.e2e_chunks > 0:
                # one call: rows uploaded in chunks, each estimated once resident
                res = cr.update_estimate(pr, chunks=a.e2e_chunks, out=mine)
            else:
                cr.update(pr)
                cr.enumerate()
                res = cr.estimate(out=mine)
            return cr.schedule_round(res)

        for _ in range(a.warmup):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        es, ee = ev(), ev()
        es.record(stream)
        for _ in range(a.steps):
            e2e_step()
        ee.record(stream)
        torch.cuda.synchronize()
        e2e_t = torch.tensor([es.elapsed_time(ee) / a.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_ms = float(e2e_t.item())
        bytes_t = torch.tensor([h2d, d2h], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(bytes_t)  # whole-job bytes: every rank's copies
        e2e = {"value": n_plans / (e2e_ms / 1e3), "unit": "cell-plans/s",
               "h2d_bytes_per_step": int(bytes_t[0]), "d2h_bytes_per_step": int(bytes_t[1]),
               "ms_per_step": e2e_ms,
               "path": ("crius_update_estimate, rows in %d pipelined chunks + round" % a.e2e_chunks
                        if world == 1 and a.e2e_chunks > 0 else
                        "update + enumerate + estimate (+ gather) + round")}

    rstats = cr.round_stats()
    sm_mhz = float(clocks.get("sm_mhz") or 1965.0)
    n_bar, floor_ms = round_floor(rstats, sm_mhz)
    round_ms = float(np.median(seg[:, 3]))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    est_roof = {"kernel": "k_estimate", "bound": "alu", "achieved": achieved_ops / 1e12,
                "peak": peak_ops / 1e12, "unit": "Tops/s", "frac": achieved_ops / peak_ops,
                "traffic": committed_traffic(workload_name(a)),
                "peak_source": f"{SM_COUNT} SMs x {INT_LANES_PER_SM} int32 lanes (ALU + FMA pipes, "
                               f"4 SMSPs x (16 + 16)) x sm_max_mhz ({src})",
                "ops_per_launch": ops * frac_units, "dp_probes": probes,
                "stage_evals": stage_evals, "share": est_ms / ms_per_step,
                "hbm": {"achieved": hbm, "peak": hbm_peak, "unit": "GB/s", "frac": hbm / hbm_peak,
                        "algorithmic_bytes_per_launch": alg_bytes,
                        "bytes_source": "SURVEY §8(d): the compute planes each unit needs + "
                                        "per-layer rows once per job + 32 B per Cell"}}
    round_roof = {"kernel": "k_round", "bound": "latency", "achieved": n_bar / (round_ms * 1e3),
                  "peak": sm_mhz / BARRIER_CYCLES, "unit": "CTA barriers/us",
                  "frac": floor_ms / round_ms, "traffic": None, "share": round_ms / ms_per_step,
                  "barrier_chain": n_bar, "floor_ms": floor_ms, "achieved_ms": round_ms,
                  "peak_source": f"{n_bar} CTA barriers (counted in the kernel) x {BARRIER_CYCLES} "
                                 f"cycles ({ROUND_THREADS}-thread __syncthreads, measured) at sm_mhz"}
    # the top-level roofline is the dominant kernel's; the other rides beside it
    dominant_round = round_ms >= est_ms
    roof = dict(round_roof if dominant_round else est_roof)
    roof["other"] = est_roof if dominant_round else round_roof
    line = {"metric": "Cell-plan evaluations/sec", "value": value, "unit": "cell-plans/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded generator, paper-shaped workloads)",
            "config": config_dict(a, pr, n_cells, n_plans, world, flush),
            "breakdown_ms": {"enumerate": float(np.median(seg[:, 0])), "estimate": est_ms,
                             "gather": float(np.median(seg[:, 2])),
                             "round": round_ms},
            "latency_ms": {"p10": float(np.percentile(step_ms, 10)),
                           "p50": float(np.median(step_ms)),
                           "p90": float(np.percentile(step_ms, 90))},
            "estimate_evals_per_s": n_plans * frac_units / (est_ms / 1e3),
            "roofline": roof,
            "round_stats": rstats,
            "clocks": clocks, "gpu_launches": int(launches)}
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and not a.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(a, W.make_config(a.config, variant=a.variant,
                                                             scale=a.scale))
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if a.json_out:
            with open(a.json_out, "w") as f:
                f.write(s + "\n")
    if xch is not None:
        xch.close()
    cr.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
