#!/usr/bin/env python
"""bench.py — DFC-Proj noisy matrix completion at BASELINE config c2 on B200.

Workload (BASELINE.json configs[1]): M = L0 + noise, m = n = 10000, r = 10,
10% of entries observed (s = 1e7, the reference generator gen_mc_instance,
P/include/dfc/simgen.hpp:45-59, seed 1), sigma = 0.1; DFC-Proj with t = 8 column blocks of
10000 x 1250 (partition seed 1, P/include/dfc/dfc.hpp:166-200) and the default ApgConfig
(P/include/dfc/solvers.hpp:19-26). Data are synthetic, seed-generated with the reference's
own generator semantics (no dataset is involved).

Metric: base-APG iterations/s ("block-iterations/s": one APG iteration of one 10000 x 1250
block = one unit). A step = one APG iteration on every block (blocks sharded over the ranks,
each advancing on its own CUDA stream). Before the W warm-up steps every block runs a fixed
prologue of --prologue iterations (default 26) so the timed window sits in the steady
rank ~700 regime that dominates a c2 solve. The reference arm (--impl reference: the oracle
port on the host cores, inputs from the oracle's own generator) runs the same prologue and
warm-up untimed and times the same iterations of block 0.
Inputs are larger than L2 (the 10k x 10k factors alone exceed 126 MB); no flush needed.

e2e: the full DFC-Proj pipeline (D step, F step, combine) through the public C ABI (host
triplets in, host estimate out, H2D/D2H inside the timed region): block-iterations/s over the
whole solve, plus the solve time and its divide / factor / combine phases.

roofline: the dominant kernel on one extra iteration of one block run alone (per-launch CUDA
events); roofline_step: all tensor-path FLOPs of the packed timed window / its device time.
"""
from __future__ import annotations

import os

# Eight solves (each with a Cholesky look-ahead helper stream) plus the normal-stream upload share
# the GPU: with the default 8 hardware work queues, streams alias onto the same queue and
# serialise against each other (measured 45-112 block-it/s run to run; 97-122 with 32 queues).
# Read when the CUDA context is created, so it is set before torch initialises CUDA.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import argparse
import json
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DFC-Proj MC solve time & base-APG iters/s at 10k×10k r=10; roofline frac"
UNIT = "block-iterations/s"
PARTITION_STREAM = 0xDFC0000000000001
FP64_DMMA_PEAK_TFLOPS = 37.1  # measured: tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak.txt)

WORKLOADS = {
    "c2": dict(m=10000, n=10000, r=10, s=10_000_000, sigma=0.1, t=8, seed=1),
    "c1": dict(m=1000, n=1000, r=10, s=200_000, sigma=0.1, t=4, seed=1),
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region: ONE long-running
    `nvidia-smi --query-gpu=... -lms 200` (the profiling recipe's clocks line), started before the
    warm-up so its NVML initialisation stays out of the timed region (spawning nvidia-smi per
    sample measured as a stall of the concurrent solves); only samples taken between mark() and
    exit are kept."""

    QUERY = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self._t0 = device, [], None
        self._proc = None
        self._reader = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self._proc.stdout:
                if self._t0 is not None and line.strip():
                    self.samples.append([x.strip() for x in line.strip().split(",")])
        except Exception:
            pass

    def start(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._reader.start()
        except Exception:
            self._proc = None
        return self

    def mark(self):
        self._t0 = time.perf_counter()

    def __enter__(self):
        self.mark()
        return self

    def __exit__(self, *a):
        time.sleep(0.25)  # at least one sample covering the end of the region
        self._t0 = None
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and "Active" in s[4 + i]
                          and "Not" not in s[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def make_blocks(P, wl):
    L0, obs = P.gen_mc_instance(wl["m"], wl["n"], wl["r"], wl["s"], wl["sigma"], wl["seed"])
    groups = P.partition_columns(wl["seed"], PARTITION_STREAM, wl["n"], wl["t"])
    blocks = [P.extract_columns(obs, g) for g in groups]
    return L0, obs, groups, blocks



def packed_shares():
    """SM-time shares of the kernels in the packed timed step, from the committed ncu launch list
    (profiles/ncu_packed_shares.json): which kernel dominates the step the value is measured on."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_packed_shares.json")) as f:
            return json.load(f)
    except Exception:
        return None


def roofline_entry(prof, peaks, peak_kind):
    ops = {k: v for k, v in prof.items() if v["launches"] > 0}
    if not ops:
        return None
    # the dominant KERNEL: the accounting splits gemm_kernel launches into >= 2 GFLOP ("gemm")
    # and smaller ("gemm_small") classes; as a kernel they are one
    kern = {k: v for k, v in ops.items() if k not in ("gemm", "gemm_small")}
    g = [ops[k] for k in ("gemm", "gemm_small") if k in ops]
    if g:
        kern["gemm_kernel"] = {f: sum(x[f] for x in g) for f in ("ms", "launches", "flops", "bytes")}
    # dominant in the PACKED timed step by SM-time (ncu launch list) when that record exists; the
    # per-launch event times below come from one block run alone (events of eight concurrent
    # streams would time each launch's wait for SMs, not the kernel)
    shares = packed_shares()
    basis = "largest event time on the lone-block step"
    cand = {k: shares[k] for k in kern if shares and isinstance(shares.get(k), (int, float))}
    if cand:
        name = max(cand, key=cand.get)
        v = kern[name]
        basis = f"largest SM-time share of the packed timed step ({cand[name]:.3f}, {shares['source']})"
    else:
        name, v = max(kern.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = v["ms"] / v["launches"]
    share = cand[name] if cand else v["ms"] / sum(x["ms"] for x in ops.values())
    if name in ("gemm_kernel", "jacobi", "cholesky", "qr_fallback"):
        achieved = v["flops"] / (v["ms"] * 1e-3) / 1e12
        peak = FP64_DMMA_PEAK_TFLOPS
        entry = dict(bound="tensor", achieved=achieved, peak=peak, unit="TFLOP/s",
                     peak_source="measured FP64 DMMA (tools/fp64_peak.cu, profiles/fp64_peak.txt)")
    else:
        achieved = v["bytes"] / (v["ms"] * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        entry = dict(bound="hbm", achieved=achieved, peak=peak, unit="GB/s",
                     peak_source=f"{peak_kind} MEASURED_PEAKS.json hbm_gbs")
    entry.update(frac=entry["achieved"] / entry["peak"], traffic=None, kernel=name, share_of_step=share,
                 dominant_by=basis,
                 launches=v["launches"], avg_launch_ms=per_launch_ms,
                 per_op={k: dict(ms=round(x["ms"], 3), launches=x["launches"],
                                 tflops=round(x["flops"] / max(x["ms"], 1e-9) / 1e9, 3),
                                 gbs=round(x["bytes"] / max(x["ms"], 1e-9) / 1e6, 1)) for k, x in ops.items()})
    traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(traffic_file):
        try:
            entry["traffic"] = json.load(open(traffic_file)).get("gemm" if name == "gemm_kernel" else name)
        except Exception:
            pass
    return entry


def nys_run(P, obs, wl):
    """DFC-Nys at the c2 shape (BASELINE configs[1]): l = d = n/t sampled columns / rows, the
    two subproblems (C-hat m x l, R-hat d x n) solved concurrently, gen_nystrom combine — the whole
    dfc_run through the C ABI, host triplets in and host factors out."""
    l = wl["n"] // wl["t"]
    t0 = time.perf_counter()
    est, info = P.dfc_run(obs, variant="nys", l=l, d=l, seed=wl["seed"], workers=2)
    wall = time.perf_counter() - t0
    its = [s.iterations for s in info["subproblems"]]
    return dict(solve_s=wall, factor_s=info["factor_ms"] / 1e3, combine_ms=info["combine_ms"], rank=est.rank,
                subproblem_iterations=its, subproblem_ranks=[s.rank for s in info["subproblems"]],
                value=sum(its) / (info["factor_ms"] * 1e-3), unit="subproblem-iterations/s",
                note=f"DFC-Nys l = d = {l}: C-hat {wl['m']}x{l} and R-hat {l}x{wl['n']} on 2 streams + gen_nystrom")


def rmf_c3(P, device):
    """BASELINE configs[2] (c3): DFC-Proj robust matrix factorisation, 10000 x 10000, r = 10, 10%
    outliers U[-10, 10], dense noise N(0, 0.01^2), t = 8 dense column blocks solved concurrently by
    apg_rmf (lambda = 1/sqrt(max(m, w)), P/include/dfc/dfc.hpp:74), column_project combine; host
    buffers in and out. Plus one profiled iteration of block 0 (the fused extrapolate / gradient /
    soft-threshold pass is the RMF's HBM kernel)."""
    m = n = 10000
    t = 8
    L0, S0, M = P.gen_rmf_instance(m, n, 10, m * n // 10, 0.01, 1, lo=-10.0, hi=1.0 * 10)
    groups = P.partition_columns(1, PARTITION_STREAM, n, t)
    blocks = [np.asfortranarray(M[:, g]) for g in groups]
    pool = ThreadPoolExecutor(max_workers=t)
    t0 = time.perf_counter()
    outs = list(pool.map(lambda b: P.apg_rmf(b, 1.0 / np.sqrt(max(b.shape)), device=device), blocks))
    f_s = time.perf_counter() - t0
    ests = [o[0] for o in outs]
    est = P.column_project(ests[0], ests, groups, device=device)
    solve_s = time.perf_counter() - t0
    its = [o[2].iterations for o in outs]
    P.prof_enable(True)
    P.apg_rmf(blocks[0], 1.0 / np.sqrt(max(blocks[0].shape)), P.ApgConfig(max_iters=1), device=device)
    prof = P.prof_collect()
    P.prof_enable(False)
    ew = prof.get("elementwise", {})
    shrink = None
    if ew.get("launches", 0) and ew["ms"] > 0:
        shrink = dict(gbs=ew["bytes"] / (ew["ms"] * 1e-3) / 1e9, launches=ew["launches"], ms=ew["ms"])
    return dict(solve_s=solve_s, factor_s=f_s, block_iterations=its, ranks=[o[2].rank for o in outs],
                value=sum(its) / f_s, unit="block-iterations/s", rank=est.rank, shrink_kernel=shrink,
                note="c3: 8 dense 10000x1250 blocks, apg_rmf concurrently on one GPU + column_project; "
                     "shrink_kernel = the fused RMF elementwise pass (algorithmic bytes / event time)")


def base_apg_window(P, obs, skip=26, win=20):
    """The metric's second half, "base-APG iters/s at 10k x 10k": the reference's Base method
    (apg_mc on the WHOLE matrix, no partition; P/include/dfc/bench.hpp:211-217) on the c2
    instance, default ApgConfig, one GPU (one subproblem, replicas only). The
    first `skip` iterations (ranks 1 -> ~3600, including the k ~ 7000 transients of iterations 14,
    25 and 26) run untimed; iterations skip+1 .. skip+win (rank ~3500 -> ~3300, every iteration
    on the dense operator 10^4 x 10^4) are timed with CUDA events, then one more iteration is
    profiled per op class."""
    import torch

    sv = P.McSolver(obs)
    t0 = time.perf_counter()
    sv.step(skip)
    torch.cuda.synchronize()
    pro_s = time.perf_counter() - t0
    w0 = P.work_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    done, tr = sv.step(win, trace=True)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    roof = step_roofline(w0, P.work_counters(), ms, max(done, 1), *measured_peaks())
    P.prof_enable(True)
    sv.step(1)
    prof = P.prof_collect()
    P.prof_enable(False)
    sv.close()
    per_op = {k: dict(ms=round(v["ms"], 2), launches=v["launches"],
                      tflops=round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 2))
              for k, v in prof.items() if v["launches"] > 0}
    return dict(value=done / (ms * 1e-3), unit="iterations/s", ms_per_iteration=ms / max(done, 1),
                window=f"iterations {skip + 1}..{skip + done} of apg_mc on the full 10000x10000 c2 matrix "
                       f"({obs.count} observations), default ApgConfig",
                ranks=[t["rank"] for t in tr], prologue_s=round(pro_s, 1),
                achieved_tflops=roof["achieved"], frac=roof["frac"], per_op_one_iteration=per_op,
                note="one subproblem: the Base method (bench.hpp:211-217); frac = tensor-path FLOPs of the window / "
                     "window device time against the measured FP64 DMMA peak")


def lowrank_window(P, block, wl, skip=60, win=20):
    import math

    import torch

    floor = wl["sigma"] * math.sqrt(wl["s"] / (wl["m"] * wl["n"])) * (
        math.sqrt(wl["m"]) + math.sqrt(block.n))
    sv = P.McSolver(block, P.ApgConfig(mu_floor=floor))
    sv.step(skip)
    torch.cuda.synchronize()
    P.prof_enable(True)
    t0 = time.perf_counter()
    done, tr = sv.step(win, trace=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    prof = P.prof_collect()
    P.prof_enable(False)
    sv.close()
    per_op = {k: dict(ms_per_it=round(v["ms"] / max(done, 1), 4), launches=v["launches"],
                      gbs=round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1))
              for k, v in prof.items() if v["launches"] > 0}
    return dict(value=done / wall, unit=UNIT, mu_floor=round(floor, 4),
                window=f"block 0, APG iterations {skip + 1}..{skip + done} under the acceptance-style floor",
                rank=tr[-1]["rank"] if tr else None, ms_per_iteration=1e3 * wall / max(done, 1), per_op=per_op,
                note="late low-rank regime: SpMM/SDDMM/elementwise rates are algorithmic bytes / event time; "
                     "kernels this small (~17 MB per SpMM) are launch- and latency-bound")


def cpu_sample(O, block, budget_s, threads, min_rank=400, max_total_s=150.0):
    """Oracle (restated reference, CPU) on one block, bounded sample of the regime the GPU
    window measures: APG iterations from the start of the solve run UNTIMED until the incoming
    rank reaches `min_rank` (the first ~6 iterations at ranks 1..400 are cheap and unlike the
    rank ~700 window), then whole iterations are timed until `budget_s` seconds of CPU work
    (or `max_total_s` overall). Returns (timed iterations, seconds, first timed iteration)."""
    O.lib().orc_set_blas_threads(threads)
    run = O.McRun(O.Observed(block.m, block.n, block.rows, block.cols, block.vals))
    t_start = time.perf_counter()
    it, rank = 0, 0
    try:
        while rank < min_rank and time.perf_counter() - t_start < max_total_s:
            tr = run.step(1)
            if not tr:
                break
            it, rank = tr[-1]["it"], tr[-1]["rank"]
        first, iters, t0 = it + 1, 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s and time.perf_counter() - t_start < max_total_s:
            if not run.step(1):
                break
            iters += 1
        dt = time.perf_counter() - t0
    finally:
        run.close()
        O.lib().orc_set_blas_threads(1)
    return iters, dt, first


def run_reference(args, wl):
    """--impl reference: the reference's CPU path on the host cores, same workload / metric /
    unit / window as the GPU arm. The C++/Eigen reference cannot be built here (Eigen3,
    GoogleTest and the vendored CLI11 are absent, no network), so this runs the oracle port
    (oracle/, a C++ restatement of P/include/dfc/*.hpp) — and only the oracle: the inputs come
    from the oracle's own restated generator / partition / extract (gen_mc_instance,
    partition_columns, extract_columns), nothing of the product package is imported.
    Window: block 0 of the c2 partition; --prologue + W untimed iterations from the start of
    the solve, then K timed iterations (each step = one APG iteration of that block) — the GPU
    arm's window, iterations prologue+W+1 .. prologue+W+K."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle as O

    threads = os.cpu_count() or 1
    L0, obs = O.gen_mc_instance(wl["m"], wl["n"], wl["r"], wl["s"], wl["sigma"], wl["seed"])
    groups = O.partition_columns(wl["seed"], PARTITION_STREAM, wl["n"], wl["t"])
    blk = O.extract_columns(obs, groups[0])
    del obs
    O.lib().orc_set_blas_threads(threads)
    run = O.McRun(blk)
    t_pro = time.perf_counter()
    run.step(args.prologue + args.warmup)
    pro_s = time.perf_counter() - t_pro
    t0 = time.perf_counter()
    tr = run.step(args.steps)
    dt = time.perf_counter() - t0
    run.close()
    done = len(tr)
    value = done / dt
    first = args.prologue + args.warmup + 1
    window = f"APG iterations {first}..{first + done - 1} of block 0 (10000x1250)"
    line = dict(impl="reference", metric=METRIC, value=value, unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * dt / max(done, 1), higher_is_better=True,
                scaling="strong", vs_baseline=None, dtype="f64",
                data="synthetic (oracle restatement of the reference generator gen_mc_instance, seed 1)",
                config=bench_config(args, wl),
                execution=dict(blocks="block 0 (10000x1250) alone: a bounded sample of the workload, the unit "
                                      "is one APG iteration on one block", window=window,
                               prologue_s=round(pro_s, 1), ranks=[t["rank"] for t in tr]),
                cpu_baseline=dict(value=value, unit=UNIT, cores=threads, kind="port",
                                  sample=f"{window}; oracle/ restatement of apg_mc (single-threaded sparse "
                                         f"ops as in the reference, OpenBLAS/LAPACK with {threads} threads)"),
                e2e=dict(value=value, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def bench_config(args, wl):
    """The `config` of the JSON line: the same dict in both arms (the reference arm measures the
    GPU arm's workload and window; what differs between the arms is under `execution`)."""
    first = args.prologue + args.warmup + 1
    return dict(workload=f"{args.workload}: DFC-Proj MC {wl['m']}x{wl['n']} r={wl['r']} "
                         f"{wl['s']} obs sigma={wl['sigma']} t={wl['t']} default ApgConfig",
                window=f"APG iterations {first}..{first + args.steps - 1} of a block (one step = one "
                       f"iteration; the unit is one iteration of one {wl['m']}x{wl['n'] // wl['t']} block)",
                l2="inputs > L2 (no flush)")


def step_roofline(w0, w1, ms, steps, peaks, peak_kind):
    """Packed-step roofline: the algorithmic work of every library op executed inside the timed
    window (always-on counters, no events) over the window's device time. Tensor-path work =
    GEMMs + Cholesky + Jacobi + Householder fallback FLOPs (FP64 DMMA); HBM-path work = the
    SDDMM / SpMM / elementwise / reduction bytes."""
    d = {k: {f: w1[k][f] - w0[k][f] for f in ("launches", "flops", "bytes")} for k in w1}
    tensor_ops = ("gemm", "gemm_small", "cholesky", "jacobi", "qr_fallback")
    fl = sum(d[k]["flops"] for k in tensor_ops)
    by = sum(d[k]["bytes"] for k in d if k not in tensor_ops)
    sec = ms * 1e-3
    ach = fl / sec / 1e12
    return dict(bound="tensor", achieved=ach, peak=FP64_DMMA_PEAK_TFLOPS, unit="TFLOP/s",
                frac=ach / FP64_DMMA_PEAK_TFLOPS, flops_per_step=fl / max(steps, 1),
                gemm_flops_per_step=(d["gemm"]["flops"] + d["gemm_small"]["flops"]) / max(steps, 1),
                hbm_bytes_per_step=by / max(steps, 1), hbm_gbs=by / sec / 1e9,
                launches_per_step=sum(v["launches"] for v in d.values()) / max(steps, 1),
                peak_source="measured FP64 DMMA (tools/fp64_peak.cu, profiles/fp64_peak.txt)",
                note="algorithmic FLOPs of all tensor-path ops in the timed window (all blocks) / window "
                     "device time (CUDA events); Jacobi FLOPs are the executed sweeps' rotation work")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--prologue", type=int, default=26)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-lowrank", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the DFC-Nys (c2) and RMF (c3) runs")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of timed CPU work for cpu_baseline")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
        return

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # DFCG_DIST_BACKEND=gloo exercises the multi-rank code path with several ranks sharing one
    # GPU (collectives on the CPU, no cross-rank kernel waits); the real runs use NCCL.
    backend = os.environ.get("DFCG_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_1107_0789_b200 as P

    peaks, peak_kind = measured_peaks()
    L0, obs, groups, blocks = make_blocks(P, wl)
    comm = None
    if dist is not None:
        # libdfcg's own transport: NCCL inside the library (the uid travels over the process
        # group), or its host-callback transport over gloo when ranks share one GPU
        from paper_1107_0789_b200.distributed import Comm, assign_blocks, dfc_run_dist

        comm = Comm.nccl(device=local) if backend == "nccl" else Comm.host()
        owner = assign_blocks([b.count for b in blocks], world)  # LPT by nnz, as dfc_run_dist assigns
    else:
        owner = [0] * wl["t"]
    mine = [g for g in range(wl["t"]) if owner[g] == rank]
    cfg = P.ApgConfig()
    solvers = {g: P.McSolver(blocks[g], cfg, device=local) for g in mine}
    pool = ThreadPoolExecutor(max_workers=max(1, len(mine)))

    trace_window = os.environ.get("DFCG_BENCH_TRACE") == "1"  # diagnostics: per-iteration host times

    def advance(n, trace=False):
        if not trace:
            return sum(pool.map(lambda g: solvers[g].step(n), mine))
        t0 = time.perf_counter()
        outs = list(pool.map(lambda g: (g, solvers[g].step(n, trace=True), time.perf_counter() - t0), mine))
        for g, (done, tr), t_end in outs:
            print(f"[window] block {g}: end {t_end * 1e3:.1f} ms, its " +
                  " ".join(f"{t['it']}:{t['ms']:.1f}/r{t['rank']}/c{t['svd_calls']}" for t in tr), file=sys.stderr)
        return sum(d for _, (d, _), _ in outs)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    advance(args.prologue)
    clocks = ClockSampler(local).start()
    for _ in range(args.warmup):
        advance(1)
    barrier()
    launches0 = P.launch_count()
    work0 = P.work_counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The K steps run back to back per block: every block's thread advances it K iterations on
    # its own stream, as the F step runs (blocks are independent, P/include/dfc/dfc.hpp:133-147);
    # a host barrier per iteration would only line the blocks' phases up against each other.
    with clocks:
        e0.record()
        iters = advance(args.steps, trace_window)
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
    launches = P.launch_count() - launches0
    work1 = P.work_counters()
    ms = e0.elapsed_time(e1)
    cdev = "cuda" if (dist is None or dist.get_backend() == "nccl") else "cpu"
    tot = torch.tensor([ms, float(iters)], dtype=torch.float64, device=cdev)
    if dist:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, iters_all = mx[0].item(), sm[1].item()
    else:
        iters_all = float(iters)
    value = iters_all / (ms * 1e-3)
    roof_step = step_roofline(work0, work1, ms, args.steps, *measured_peaks())

    # kernel accounting on one extra iteration of one block, run alone (outside the timed
    # region) so every op's CUDA-event interval is its own device time
    torch.cuda.synchronize()
    P.prof_enable(True)
    solvers[mine[0]].step(1)
    prof = P.prof_collect()
    P.prof_enable(False)
    roof = roofline_entry(prof, peaks, peak_kind)
    # the tensor-core GEMMs (>= 2 GFLOP: the operator products, CholQR Grams / triangular
    # products, the left factor) of that step, against the FP64 DMMA roofline
    g = prof.get("gemm", {})
    roof_gemm = None
    if g.get("launches", 0) > 0 and g["ms"] > 0:
        ach = g["flops"] / (g["ms"] * 1e-3) / 1e12
        roof_gemm = dict(bound="tensor", achieved=ach, peak=FP64_DMMA_PEAK_TFLOPS, unit="TFLOP/s",
                         frac=ach / FP64_DMMA_PEAK_TFLOPS, launches=g["launches"],
                         avg_launch_ms=g["ms"] / g["launches"], kernel="gemm_kernel (DMMA m8n8k4)")

    # combine on the current block estimates (column_project, P/include/dfc/sketch.hpp:170-199);
    # at N > 1 the combine runs inside dfc_run_dist (e2e below: basis broadcast + row gather)
    combine_ms, combine_ops = None, None
    if dist is None:
        ests = {g: solvers[g].finish()[0] for g in mine}
        barrier()
        P.prof_enable(True)
        t0 = time.perf_counter()
        P.column_project(ests[0], [ests[g] for g in range(wl["t"])], groups, device=local)
        barrier()
        combine_ms = 1e3 * (time.perf_counter() - t0)
        cprof = P.prof_collect()
        P.prof_enable(False)
        combine_ops = {k: dict(ms=round(v["ms"], 3), launches=v["launches"],
                               tflops=round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3))
                       for k, v in cprof.items() if v["launches"] > 0}
    for sv in solvers.values():
        sv.close()

    # e2e: the full DFC-Proj pipeline through the public C ABI, D step included
    # (P/include/dfc/dfc.hpp:166-200: partition + extract, F, combine; DfcReport.total_ms covers
    # all three): host triplets in, host factors out. N = 1: one dfcg_dfc_run call. N > 1: every
    # rank partitions, extracts its own blocks, solves them and joins the distributed combine.
    e2e = None
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        if dist is None:
            est, info = P.dfc_run(obs, "proj", t=wl["t"], seed=wl["seed"], workers=wl["t"], device=local)
            tot_iters = float(sum(r.iterations for r in info["subproblems"]))
            h2d = obs.count * 24
            d2h = (est.left.size + est.right.size) * 8
            phases = dict(divide_ms=info["divide_ms"], factor_ms=info["factor_ms"], combine_ms=info["combine_ms"],
                          total_ms=info["total_ms"])
        else:
            # every rank: the whole observation set in, its LPT share solved, the combine's
            # exchange over libdfcg's communicator, the final estimate out (dfcg_dfc_run_dist)
            est, info = dfc_run_dist(obs, comm, "proj", t=wl["t"], seed=wl["seed"], workers=max(1, len(mine)),
                                     device=local)
            tot_iters = float(sum(r.iterations for r in info["subproblems"]))
            h2d = obs.count * 24
            d2h = (est.left.size + est.right.size) * 8
            phases = dict(divide_ms=info["divide_ms"], factor_ms=info["factor_ms"], combine_ms=info["combine_ms"],
                          total_ms=info["total_ms"], owner=info["owner"])
            combine_ms = info["combine_ms"]
        barrier()
        wall = time.perf_counter() - t0
        wt = torch.tensor([wall], dtype=torch.float64, device=cdev)
        if dist:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        wall = wt.item()
        e2e = dict(value=tot_iters / wall, unit=UNIT, h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                   dfc_proj_solve_s=wall, block_iterations=int(tot_iters), **phases,
                   note="one e2e step = the whole DFC-Proj pipeline (D: partition + extract, F: all blocks to "
                        "convergence, C: column_project) through the C ABI from host triplets to host factors")

    # Secondary regime ("report both regimes"): the acceptance-style floor
    # (P/tests/acceptance.cpp:127-130) drives block 0 to its low-rank tail, where the sparse
    # kernels are the per-iteration work. One block, iterations 61..80, per-op rates.
    lowrank = None
    if rank == 0 and not args.no_lowrank:
        lowrank = lowrank_window(P, blocks[0], wl)

    # the other BASELINE F-step configurations on this GPU (rank 0, N = 1): base APG on the
    # whole matrix, DFC-Nys at c2, c3
    nys = rmf = base = None
    if rank == 0 and world == 1 and not args.no_extra and args.workload == "c2":
        base = base_apg_window(P, obs)
        nys = nys_run(P, obs, wl)
        rmf = rmf_c3(P, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle as O

        threads = os.cpu_count() or 1
        done, dt, first = cpu_sample(O, blocks[0], args.cpu_budget, threads)
        cpu = dict(value=done / max(dt, 1e-9), unit=UNIT, cores=threads, kind="port",
                   sample=f"block 0 (10000x1250): APG iterations {first}..{first + done - 1} ({dt:.1f} s), the "
                          f"first iterations entered at rank >= 400 (earlier, cheaper iterations run untimed); "
                          f"oracle/ restatement of apg_mc (single-threaded sparse ops as in the reference, "
                          f"OpenBLAS/LAPACK with {threads} threads)")

    if rank == 0:
        line = dict(metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=ms / max(args.steps, 1), higher_is_better=True, scaling="strong", vs_baseline=None,
                    dtype="f64", data="synthetic (reference generator gen_mc_instance, seed 1)",
                    config=bench_config(args, wl),
                    execution=dict(blocks="every block", blocks_per_gpu=len(mine),
                                   parallelism=f"{wl['t']} blocks over {world} GPU(s) (LPT by nnz), one CUDA "
                                               f"stream per block; combine over libdfcg's "
                                               f"{'NCCL' if backend == 'nccl' or world == 1 else 'host'} transport"),
                    roofline=roof, roofline_step=roof_step, roofline_gemm=roof_gemm, cpu_baseline=cpu, e2e=e2e, gpu_launches=int(launches),
                    clocks=clocks.summary(), combine_ms=combine_ms,
                    combine=dict(ms=combine_ms, device_ops=combine_ops,
                                 note="DFC-Proj column_project of the 8 block estimates (N = 1: host factors in and "
                                      "out, device_ops = CUDA-event time per op class; N > 1: the combine phase of "
                                      "dfc_run_dist, basis broadcast + projected-row gather)"),
                    lowrank=lowrank, base_apg=base, nys_c2=nys, rmf_c3=rmf)
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
