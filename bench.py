#!/usr/bin/env python
"""AIDW hot-path benchmark.

One step = the whole hot path (S1 kNN + r_obs, S3 allreduce of the R bounds when
N > 1, S4 alpha, S5 weighting pass) over one batch of queries whose data and
queries are already resident in HBM.

  --config C4 (default): 1,024,000 data x 1,024,000 queries, k = 10, fp32, uniform,
          GLOBAL R bounds (BASELINE.json configs[3], the metric's 1M x 1M configuration)
  --config C5: 1,024,000 data x 8,192,000 grid queries (configs[4])
  N > 1 : strong scaling (default): the job's queries are split into contiguous rank
          blocks [r nq/N, (r+1) nq/N) -- BASELINE C4 "1 GPU vs 8 GPUs query-sharded",
          C5 "2/4/8 GPU scaling" -- with data replicated and the GLOBAL bounds joined
          by one NCCL allreduce(MAX) per step; --scaling weak gives every rank nq queries.

The fp32 line carries an ``fp64`` sub-record (the metric's fp64 point, same workload
and launch configuration), ``e2e`` (aidw_run_host from pinned host queries) and
``e2e_full`` (aidw_create from pinned host data + the e2e step + destroy).

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the
"reference arm" of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

ND = 1000 * datagen.K_SIZE
NQ_PER_GPU = 1000 * datagen.K_SIZE
K_NN = 10
SEED = 1004  # C4
BENCH_CONFIGS = ("C4", "C5")  # the BASELINE configs whose data fill one GPU and whose queries shard


def metric_name(cfg="C4", dtype="f32"):
    prec = "fp64" if dtype == "f64" else "fp32"
    q = "1M queries" if cfg == "C4" else "8.19M grid queries"
    return f"AIDW interpolated points/sec ({prec}; {cfg}: 1M data x {q}, k=10, GLOBAL R bounds)"


METRIC = metric_name()
# Roofline model of the weighting pass.  Per (query, data point) pair
# the method needs 7 FP32 operations (s: 2 sub + mul + fma; exponent fma; two sums)
# and 2 transcendentals (log2, exp2).  A transcendental costs 1 SFU op, or 8 FMA-pipe
# ops when evaluated as a polynomial; the best split of the work over the two pipes
# gives the bound.  Pipe rates: profiles/r01_pipe_peaks.json (measured on B200; re-measured
# in round 2, profiles/r02_pipe_peaks.jsonl: MUFU 15.94, FFMA2 122.8 FMA/clk/SM, DFMA 62.7,
# MUFU.RCP 15.90 -- within 0.9 %).
WEIGHT_FP32_PER_PAIR = 7
TRANSC_PER_PAIR = 2
POLY_FMA_PER_TRANSC = 8
MUFU_PER_CLK_SM = 15.96   # measured MUFU.EX2/LG2 per SM per clock
FMA_PER_CLK_SM = 123.2    # measured FFMA2 (packed) FMA ops per SM per clock
N_SM = 148
# fp64 (--dtype f64): the weighting pass has no hardware transcendental;
# per pair the kernel issues 21 FP64 operations (round 2: distance 4, table + degree-3
# log2 6, exponent 1, table + degree-4 exp2 8, sums 2; round 1 issued 25 with degree-5
# polynomials, profiles/archive_r01/r01_ncu_interp_f64_v12.json) on the FP64 pipe; DFMA rate
# measured by tools/pipe_peaks.cu (profiles/r01_pipe_peaks.json).
DP_PER_PAIR = 21
DFMA_PER_CLK_SM = 63.23  # measured (profiles/r01_pipe_peaks.json dfma_per_clk_sm)
# The algorithmic fp64 bound: FP64 ops per pair that evaluate Eq. 1 to
# the north star's fp64 tolerance (1e-10 relative) -- distance 4, log2 with a 256-entry
# table and a degree-3 polynomial (error 2^-36) 5, exponent 1, exp2 with a 64-entry table
# and a degree-4 polynomial 8, two sums 2.
DP_ALGO_PER_PAIR = 20
KNN_FILTER_FMA_PER_PAIR = 2  # the r01 fp32 filter t = pp + a cx + b cy: 2 FMA per pair (one FFMA2 per couple)
KNN_STRIP_FMA_PER_PAIR = 1   # round 2: the strip pre-test t1 = ps + A u, ONE fp16 FMA per pair (HFMA2: 2 per lane
                             # per issue, the FFMA2 cadence) -- the least any exact brute-force pass can spend


def weight_clk_per_pair(fp32=WEIGHT_FP32_PER_PAIR, transc=TRANSC_PER_PAIR):
    """min over the SFU fraction of max(FMA-pipe time, SFU time), clocks per pair per SM."""
    best = None
    for i in range(0, 2001):
        f = transc * i / 2000.0  # transcendentals moved to the FMA pipe
        t = max((fp32 + POLY_FMA_PER_TRANSC * f) / FMA_PER_CLK_SM, (transc - f) / MUFU_PER_CLK_SM)
        best = t if best is None else min(best, t)
    return best


# Exact-exponent classes: a query whose alpha is exactly 1, 2 or 3 (and
# whose d1^2 is in range) needs one transcendental per pair -- rsqrt, rcp or rsqrt^3 --
# and s (4) + the two sums (2) [+ 2 FMUL for the cube] FP32 ops.
CLASS_OPS = {"general": (WEIGHT_FP32_PER_PAIR, TRANSC_PER_PAIR), "a1": (6, 1), "a2": (6, 1), "a3": (8, 1)}


def class_fractions(alpha, d1sq):
    """Fraction of queries per weighting class (same rule as passes.cuh alpha_class)."""
    ok = (d1sq >= 2.0 ** -78) & (d1sq <= 2.0 ** 66)
    n = max(1, alpha.numel())
    fr = {c: float(((alpha == v) & ok).sum()) / n for c, v in (("a1", 1.0), ("a2", 2.0), ("a3", 3.0))}
    fr["general"] = 1.0 - sum(fr.values())
    return fr


def weight_clk_mix(fr):
    return sum(f * weight_clk_per_pair(*CLASS_OPS[c]) for c, f in fr.items())


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"sm_max_mhz": 1965.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 7:
                self.rows.append(p)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_oracle_rate(x, y, z, qx, qy, k=K_NN, target_s=12.0):
    """Time the oracle as it stands (all host cores) on a bounded query sample of the
    workload; returns (points/s, cores, sample description)."""
    import oracle
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    cores = oracle.num_threads()
    # calibrate with a small sample, then size the sample for ~target_s seconds
    n0 = max(cores, 16)
    t0 = time.perf_counter()
    _oracle_steps(oracle, x, y, z, qx[:n0], qy[:n0], k)
    dt0 = time.perf_counter() - t0
    n = int(min(len(qx), max(n0, n0 * target_s / max(dt0, 1e-3))))
    n = max(cores, (n // cores) * cores)
    t0 = time.perf_counter()
    _oracle_steps(oracle, x, y, z, qx[:n], qy[:n], k)
    dt = time.perf_counter() - t0
    return n / dt, cores, f"{n} of {len(qx)} queries x all {len(x)} data points, full AIDW (kNN + alpha + Eq. 1), fp64"


def cpu_single_thread():
    """The paper-comparable CPU row (sequential double): the oracle on ONE
    core over the whole of C1 and C2."""
    import oracle
    prev = oracle.num_threads()
    oracle.set_num_threads(1)
    out = {}
    try:
        for c in ("C1", "C2"):
            cfg = datagen.CONFIGS[c]
            x, y, z = datagen.make_data(c)
            qx, qy = datagen.make_queries(c)
            t0 = time.perf_counter()
            _oracle_steps(oracle, x, y, z, qx, qy, cfg["k"])
            dt = time.perf_counter() - t0
            out[c] = {"seconds": dt, "points_per_s": len(qx) / dt, "pair_evals_per_s": 2.0 * len(qx) * len(x) / dt,
                      "nd": len(x), "nq": len(qx), "k": cfg["k"]}
    finally:
        oracle.set_num_threads(prev)
    return out


def _oracle_steps(oracle, x, y, z, qx, qy, k=K_NN):
    re = oracle.r_exp(len(x), oracle.bbox_area(x, y))
    robs = oracle.knn_f64(x, y, qx, qy, k)
    rmin, rmax = oracle.r_bounds(robs, re, oracle.GLOBAL)
    a = oracle.alpha(robs, re, datagen.ALPHA_LEVELS, rmin, rmax)
    return oracle.idw(x, y, z, qx, qy, a)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def job_queries(cfg, q0, n):
    """Queries [q0, q0 + n) of the config's query stream (uniform: counter-based draws at
    any offset; C5: the grid in row-major order)."""
    return datagen.make_queries(cfg, nq=n, offset=q0)


def job_nq(cfg, nq_arg):
    return nq_arg if nq_arg else datagen.CONFIGS[cfg]["nq"]


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = args.config
    x, y, z = datagen.make_data(cfg)
    nq_total = job_nq(cfg, args.nq) * (args.gpus if args.scaling == "weak" else 1)
    qx, qy = job_queries(cfg, 0, nq_total)
    import oracle
    oracle.build()
    # rank 0 runs alone: use every host core it may run on (torchrun sets OMP_NUM_THREADS=1)
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    cores = oracle.num_threads()
    # each step: a bounded sample sized so the whole run ends within minutes
    per_step = max(cores, int(args.ref_queries_per_step or 32 * cores))
    times = []
    for i in range(args.warmup + args.steps):
        s = (i * per_step) % (len(qx) - per_step)
        t0 = time.perf_counter()
        _oracle_steps(oracle, x, y, z, qx[s:s + per_step], qy[s:s + per_step])
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = per_step / (ms / 1e3)
    sample = f"{per_step} queries per step x all {len(x)} data points, full AIDW (kNN + alpha + Eq. 1), fp64"
    out = {
        "impl": "reference", "metric": metric_name(cfg), "value": value, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.gpus, nq_total, args.scaling), "nd": len(x), "k": K_NN,
                   "nq_total": nq_total},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def query_block(rank, world, nq, strong):
    """This rank's queries as (first index, count, job total): weak scaling gives every rank
    ``nq`` queries; strong scaling splits ``nq`` into contiguous blocks [r nq/N, (r+1) nq/N)
    (SURVEY §8(e)), so the ranks' blocks concatenate to the 1-GPU batch."""
    if strong:
        q0 = rank * nq // world
        return q0, (rank + 1) * nq // world - q0, nq
    return rank * nq, nq, nq * world


def workload_name(cfg, n, nq_total, scaling="strong", mode="global", dtype="f32"):
    rb = {"global": "GLOBAL R bounds", "fixed": "FIXED R bounds (0, 2), fused kernel",
          "fixed3": "FIXED R bounds (0, 2), stage kernels"}[mode]
    prec = "fp64" if dtype == "f64" else "fp32"
    qd = "uniform queries" if datagen.CONFIGS[cfg]["queries"] == "uniform" else "grid queries (4096 x 2000)"
    std = nq_total == datagen.CONFIGS[cfg]["nq"]
    tag = cfg if std else f"{cfg}-shaped"
    s = f"{tag}: 1,024,000 uniform data x {nq_total:,} {qd}, k=10, {prec}, {rb}"
    if n > 1:
        per = nq_total // n
        s += (f"; strong-scaled over {n} GPUs (~{per:,} queries each)" if scaling == "strong" else
              f"; weak-scaled, {per:,} queries per GPU")
        if mode == "global":
            s += ", bounds allreduced"
    return s


def time_steps(step, steps, st, flush, group):
    """Run ``steps`` timed steps (CUDA events on the launching stream, L2 flushed between
    steps outside the events); returns the per-phase ms array [steps, 4]."""
    import torch
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush.fill_(i & 0xFF)  # L2 flush (256 MiB write) outside the step's events
        step(evs[i])
    torch.cuda.synchronize()
    return np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(4)] for i in range(steps)])


def max_over_ranks(v, group, dev):
    if group is None:
        return float(v)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class PathRunner:
    """One precision of the hot path on this rank's query block, resident in HBM."""

    def __init__(self, P, cfg, x, y, z, qx_np, qy_np, tdt, gpu, dev, mode, exchange, group):
        import torch
        self.P, self.mode, self.exchange, self.group = P, mode, exchange, group
        self.tdt, self.dev = tdt, dev
        self.eng = P.AIDW(x, y, z, dtype=tdt, device=gpu)
        self.qx = torch.as_tensor(qx_np, dtype=tdt, device=dev)
        self.qy = torch.as_tensor(qy_np, dtype=tdt, device=dev)
        self.nq = self.qx.numel()
        if exchange:  # device-side bounds exchange over peer memory
            from paper_1511_02186_b200.partition import connect_exchange
            connect_exchange(self.eng, group)
        self.r_obs = torch.empty(self.nq, dtype=tdt, device=dev)
        self.d1 = torch.empty_like(self.r_obs)
        self.al = torch.empty_like(self.r_obs)
        self.zo = torch.empty_like(self.r_obs)
        self.mm = torch.empty(2, dtype=tdt, device=dev)
        self.st = torch.cuda.current_stream(dev)

    def step(self, ev=None):
        from paper_1511_02186_b200.partition import allreduce_bounds
        P, st, lv, e = self.P, self.st, datagen.ALPHA_LEVELS, self.eng
        if ev: ev[0].record(st)
        if self.mode == "fixed":  # N1: one fused launch
            P.aidw_run_fixed(e.h, self.qx, self.qy, K_NN, lv, 0.0, 2.0, P.NORMALIZED, self.zo, None, None, st)
            for i in range(1, 5):
                if ev: ev[i].record(st)
            return
        P.aidw_knn_robs(e.h, self.qx, self.qy, K_NN, self.r_obs, self.d1, self.mm, None, st)
        if ev: ev[1].record(st)
        if self.group is not None and self.mode == "global" and not self.exchange:
            allreduce_bounds(self.mm, self.group)
        if ev: ev[2].record(st)
        if self.mode == "fixed3":
            P.aidw_alpha(e.h, self.r_obs, lv, P.FIXED, 0.0, 2.0, self.mm, P.NORMALIZED, self.al, st)
        else:  # with --exchange p2p the alpha kernel reads the peers' pushed bounds (mm = NULL)
            P.aidw_alpha(e.h, self.r_obs, lv, P.GLOBAL, 0.0, 0.0, None if self.exchange else self.mm, P.NORMALIZED,
                         self.al, st)
        if ev: ev[3].record(st)
        P.aidw_interpolate(e.h, self.qx, self.qy, self.al, self.d1, self.zo, st)
        if ev: ev[4].record(st)

    def timed(self, steps, warmup, flush):
        """W warm-up steps, then K timed steps bracketed by a barrier and a synchronize on
        both sides; returns (per-phase ms [K, 4], max-over-ranks ms per step, launches)."""
        import torch
        import torch.distributed as dist
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        l0 = self.eng.launches
        if self.group is not None:
            dist.barrier(self.group)
        torch.cuda.synchronize()
        per = time_steps(self.step, steps, self.st, flush, self.group)
        if self.group is not None:
            dist.barrier(self.group)
        if self.exchange:
            self.eng.check()  # a timed-out peer wait is reported, never silently used
        launches = self.eng.launches - l0
        return per, max_over_ranks(per.sum(1).mean(), self.group, self.dev), launches


def e2e_step(P, eng, hx, hy, hz, dev, mode, exchange, group):
    """One public-API step from pinned host queries to pinned host Z."""
    lv = datagen.ALPHA_LEVELS
    if mode in ("fixed", "fixed3") or group is not None or exchange:
        dx = hx.to(dev, non_blocking=True)
        dy = hy.to(dev, non_blocking=True)
        if mode == "fixed":
            zz = eng.run_fixed(dx, dy, K_NN, lv, 0.0, 2.0)
        elif mode == "fixed3":
            zz = eng.run(dx, dy, K_NN, lv, P.FIXED, 0.0, 2.0)
        else:
            zz = eng.run(dx, dy, K_NN, lv, P.GLOBAL, group=group)
        hz.copy_(zz, non_blocking=True)
    else:
        eng.run_host(hx, hy, K_NN, lv, P.GLOBAL, out=hz)  # C ABI aidw_run_host


def e2e_api_name(mode, exchange, group):
    return ("aidw_run_fixed + torch H2D/D2H (pinned)" if mode == "fixed" else
            "AIDW.run(FIXED) + torch H2D/D2H (pinned)" if mode == "fixed3" else
            "aidw_run_host (C ABI, pinned host buffers)" if group is None and not exchange else
            "AIDW.run + torch H2D/D2H (pinned), device-side bounds exchange" if exchange else
            "AIDW.run + torch H2D/D2H (pinned), allreduce")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=BENCH_CONFIGS,
                    help="C4: 1M x 1M uniform (default); C5: 1M data x 8.19M grid queries")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f64", action="store_true", help="skip the fp64 sub-record")
    ap.add_argument("--f64-steps", type=int, default=3)
    ap.add_argument("--profile", action="store_true", help="minimal run for ncu (no baselines, no flush)")
    ap.add_argument("--nq", type=int, default=0,
                    help="queries in total (strong, default: the config's) or per GPU (--scaling weak)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the config's queries split into contiguous rank blocks "
                         "[r nq/N, (r+1) nq/N) (BASELINE C4 1 vs 8 GPUs, C5 2/4/8); weak: --nq per GPU")
    ap.add_argument("--ref-queries-per-step", type=int, default=0)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="GLOBAL bounds: NCCL allreduce(MAX) (default) or the device-side push over "
                         "peer memory (aidw_exchange_*, no collective per step)")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                    help="working precision of the main line (f64: the fp64 point of the metric)")
    ap.add_argument("--mode", default="global", choices=["global", "fixed", "fixed3"],
                    help="global: 3 kernels + allreduce (north star, default); fixed: R bounds (0, 2), "
                         "one fused kernel per step (N1); fixed3: R bounds (0, 2) on the stage kernels")
    args = ap.parse_args()
    if args.scaling == "weak" and args.config != "C4":
        raise SystemExit("--scaling weak draws fresh uniform queries per rank: C4 only")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1511_02186_b200 as P

    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    # one process per GPU; AIDW_DIST_BACKEND=gloo + more ranks than GPUs is a logic
    # test mode (ranks share a device), never a bench configuration
    backend = os.environ.get("AIDW_DIST_BACKEND", "nccl")
    gpu = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    group = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD

    cfg = args.config
    strong = args.scaling == "strong"
    q0, nq, nq_total = query_block(rank, world, job_nq(cfg, args.nq), strong)
    f64 = args.dtype == "f64"
    if f64 and args.mode == "fixed":
        raise SystemExit("--mode fixed (the fused kernel) is fp32 only; use fixed3 for fp64")
    tdt = torch.float64 if f64 else torch.float32
    x, y, z = datagen.make_data(cfg)
    nd = len(x)
    qx_np, qy_np = job_queries(cfg, q0, nq)
    flush = None if args.profile else torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    exchange = args.exchange == "p2p" and args.mode == "global"
    run = PathRunner(P, cfg, x, y, z, qx_np, qy_np, tdt, gpu, dev, args.mode, exchange, group)

    if args.profile:
        for _ in range(args.warmup):
            run.step()
        torch.cuda.synchronize()
        run.step()
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile_run": True, "nq": nq}))
        return 0

    with ClockSampler(gpu) as clk:
        per, ms, launches = run.timed(args.steps, args.warmup, flush)
    zs = run.zo[:8].cpu()
    assert torch.isfinite(zs).all()
    d1_cls, al_cls = run.d1, run.al
    tb = 8 if f64 else 4

    # ---- e2e: public API from pinned host buffers, H2D + D2H inside the timed region
    e2e = e2e_full = None
    if not args.no_e2e:
        hx = torch.as_tensor(qx_np, dtype=tdt).pin_memory()
        hy = torch.as_tensor(qy_np, dtype=tdt).pin_memory()
        hz = torch.empty(nq, dtype=tdt).pin_memory()
        e2e_steps = max(1, min(args.steps, 3))
        if group is not None:
            dist.barrier()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(e2e_steps):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(run.st)
            e2e_step(P, run.eng, hx, hy, hz, dev, args.mode, exchange, group)
            e1.record(run.st)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        e2e_ms = max_over_ranks(tot / e2e_steps, group, dev)
        e2e = {"value": nq_total / (e2e_ms / 1e3), "unit": "points/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": 2 * tb * nq_total, "d2h_bytes_per_step": tb * nq_total,
               "api": e2e_api_name(args.mode, exchange, group)}
        # e2e_full: the data upload and S0 (aidw_create from pinned host
        # data: H2D, repack, bbox, Eq. 2, Morton order) + the step above + aidw_destroy
        if not exchange:
            hdata = torch.stack([torch.as_tensor(v, dtype=tdt) for v in (x, y, z)]).contiguous().pin_memory()
            full_steps = max(1, min(args.steps, 2))
            tot = 0.0
            for i in range(full_steps):
                flush.fill_(i & 0xFF)
                torch.cuda.synchronize()
                if group is not None:
                    dist.barrier()
                t0 = time.perf_counter()
                eng2 = P.AIDW.from_host(hdata, device=gpu)  # aidw_create from pinned host data
                e2e_step(P, eng2, hx, hy, hz, dev, args.mode, False, group)
                torch.cuda.synchronize()
                eng2.close()  # aidw_destroy
                tot += time.perf_counter() - t0
            full_ms = max_over_ranks(1e3 * tot / full_steps, group, dev)
            e2e_full = {"value": nq_total / (full_ms / 1e3), "unit": "points/s", "ms_per_step": full_ms,
                        "h2d_bytes_per_step": 3 * tb * nd * world + 2 * tb * nq_total,
                        "d2h_bytes_per_step": tb * nq_total,
                        "api": "aidw_create (pinned host data) + " + e2e["api"] + " + aidw_destroy; host wall clock"}

    # ---- the metric's fp64 point on the same workload (sub-record)
    f64_rec = None
    if not f64 and not args.no_f64 and args.mode == "global":
        del run
        torch.cuda.empty_cache()
        r64 = PathRunner(P, cfg, x, y, z, qx_np, qy_np, torch.float64, gpu, dev, "global", exchange, group)
        per64, ms64, l64 = r64.timed(args.f64_steps, 3, flush)
        f64_rec = fp64_record(per64, ms64, nq, nq_total, nd, l64, peaks())
        del r64

    if rank != 0:
        dist.destroy_process_group()
        return 0

    pk = peaks()
    clocks = clk.summary()
    f_max = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    pairs = float(nq) * nd
    knn_ms = float(per[:, 0].mean())
    ar_ms = float(per[:, 1].mean())
    alpha_ms = float(per[:, 2].mean())
    interp_ms = float(per[:, 3].mean())
    # dominant kernel: the weighting pass, bound by the SFU + FMA pipes together
    interp_rate = pairs / (interp_ms / 1e3)
    fr = (class_fractions(al_cls, d1_cls) if args.mode != "fixed" and not f64 else
          {"general": 1.0, "a1": 0.0, "a2": 0.0, "a3": 0.0})
    w_clk = weight_clk_mix(fr)
    sfu_peak_pairs = N_SM * f_max / w_clk
    path_clk_per_pair = KNN_STRIP_FMA_PER_PAIR / FMA_PER_CLK_SM + w_clk
    path_peak_pairs = N_SM * f_max / path_clk_per_pair
    traffic = knn_traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tr.get("interp_dram_bytes_per_launch")
        knn_traffic = tr.get("knn_dram_bytes_per_launch")
    except Exception:
        pass
    value = nq_total / (ms / 1e3)
    phases = {"knn_robs": knn_ms, "allreduce": ar_ms, "alpha": alpha_ms, "interpolate": interp_ms}
    if args.mode == "fixed":  # one fused kernel per step: its roofline is the path bound
        fused_rate = pairs / (knn_ms / 1e3)
        roof = {"bound": "alu", "kernel": "fused_fixed_kernel (N1: S1..S5 in one launch)",
                "achieved": fused_rate / 1e9, "peak": path_peak_pairs / 1e9, "unit": "Gpair/s",
                "frac": fused_rate / path_peak_pairs, "traffic": None,
                "peak_basis": "kNN 1 FMA/pair (the strip pre-test) on the FMA pipe + the pipe-balanced weighting bound "
                              f"({w_clk:.4f} clk/pair), {N_SM} SM x {f_max / 1e6:.0f} MHz"}
        phases = {"fused": knn_ms}
    elif f64:
        roof = fp64_roofline(interp_ms, pairs, f_max, clocks)
    else:
        roof = {
            "bound": "alu", "kernel": "interp_f32x2_kernel (S5 weighting pass)",
            "achieved": interp_rate / 1e9, "peak": sfu_peak_pairs / 1e9, "unit": "Gpair/s",
            "frac": interp_rate / sfu_peak_pairs, "traffic": traffic,
            "peak_basis": f"{N_SM} SM x {f_max / 1e6:.0f} MHz / {w_clk:.4f} clk per pair: 7 FP32 + 2 "
                          f"transcendentals per pair (exact-exponent classes: 6-8 FP32 + 1) split optimally "
                          f"between SFU ({MUFU_PER_CLK_SM}/clk) and FMA pipe ({FMA_PER_CLK_SM}/clk, 8 ops per "
                          f"polynomial transcendental), weighted by the class mix; measured pipe rates "
                          f"profiles/r01_pipe_peaks.json (r02 re-measure: profiles/r02_pipe_peaks.jsonl); sm_max_mhz from MEASURED_PEAKS.json",
            "class_mix": {c: round(f, 5) for c, f in fr.items()},
            "hbm_gb_per_s": (traffic / (interp_ms / 1e3) / 1e9) if traffic else None,
            "general_clk_per_pair": weight_clk_per_pair(),
            "sfu_only_peak": N_SM * MUFU_PER_CLK_SM / TRANSC_PER_PAIR * f_max / 1e9,
            "path_frac": (pairs / (ms / 1e3)) / path_peak_pairs,
            "path_peak_basis": "kNN 1 FMA/pair (the strip pre-test, DESIGN.md 4.1) on the FMA pipe + the weighting "
                               "bound above, per SM",
            "frac_at_measured_clock": (interp_rate / sfu_peak_pairs) * (f_max / (clocks["sm_mhz"] * 1e6))
            if clocks.get("sm_mhz") else None,
            "knn": knn_roofline(knn_ms, pairs, f_max, knn_traffic),
        }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, cores, sample = cpu_oracle_rate(x, y, z, qx_np, qy_np)
        cpu = {"value": rate, "unit": "points/s", "cores": cores, "kind": "oracle", "sample": sample,
               "cpu_model": cpu_model(), "single_thread": cpu_single_thread()}
    out = {
        "metric": metric_name(cfg, args.dtype),
        "value": value,
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": workload_name(cfg, world, nq_total, args.scaling, args.mode, args.dtype),
                   "nd": nd, "nq_per_gpu": nq, "nq_total": nq_total,
                   "k": K_NN, "alpha_levels": list(datagen.ALPHA_LEVELS),
                   "rbounds": {"global": "global", "fixed": "fixed (0, 2), fused single kernel",
                               "fixed3": "fixed (0, 2), stage kernels"}[args.mode],
                   "mu": "normalized",
                   "l2": "flushed between steps (256 MiB write outside the timed events)",
                   "parallelism": f"query-sharded x{world} ({args.scaling}), data replicated",
                   "bounds_exchange": ("device push over peer memory (aidw_exchange_*)" if exchange else
                                       "NCCL allreduce(MAX)" if world > 1 else "local")},
        "pair_evals_per_s": 2.0 * nq_total * nd / (ms / 1e3),
        "aidw_pairs_per_s": float(nq_total) * nd / (ms / 1e3),
        "phases_ms": phases,
        "roofline": roof,
        "fp64": f64_rec,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_full": e2e_full,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    print(json.dumps(out), flush=True)
    if group is not None:
        dist.destroy_process_group()
    return 0


def knn_roofline(knn_ms, pairs, f_max, traffic=None):
    """kNN kernel against its FMA-pipe bound.  Since round 2 every pair is
    touched by the strip pre-test t1 = ps + A u, one fp16 FMA per pair (HFMA2 carries two
    per lane at the FFMA2 cadence), so the bound is ONE FMA per pair -- one arithmetic
    operation per pair, the least an exact brute-force pass can do.  `frac_vs_fp32_filter`
    keeps the round-1 bound (the fp32 filter's 2 FMA per pair) for comparison."""
    rate = pairs / (knn_ms / 1e3)
    peak = N_SM * f_max * FMA_PER_CLK_SM / KNN_STRIP_FMA_PER_PAIR
    peak_r01 = N_SM * f_max * FMA_PER_CLK_SM / KNN_FILTER_FMA_PER_PAIR
    return {"kernel": "knn_filter_kernel (S1+S2 kNN pass)", "bound": "alu", "achieved": rate / 1e9,
            "peak": peak / 1e9, "unit": "Gpair/s", "frac": rate / peak, "traffic": traffic,
            "peak_basis": f"{N_SM} SM x {f_max / 1e6:.0f} MHz x {FMA_PER_CLK_SM} FMA lanes/clk / "
                          f"{KNN_STRIP_FMA_PER_PAIR} FMA per pair (strip pre-test t1 = ps + A u, fp16, DESIGN.md 4.1)",
            "frac_vs_fp32_filter": rate / peak_r01,
            "fp32_filter_basis": f"{KNN_FILTER_FMA_PER_PAIR} FMA per pair (t = pp + a cx + b cy; the round-1 bound)"}


def fp64_roofline(interp_ms, pairs, f_max, clocks):
    """fp64 weighting pass against the FP64-pipe bound of DESIGN.md §4.9: the minimum
    FP64 operation count per pair that evaluates Eq. 1 within the north star's 1e-10."""
    rate = pairs / (interp_ms / 1e3)
    peak = N_SM * f_max * DFMA_PER_CLK_SM / DP_ALGO_PER_PAIR
    return {"bound": "alu", "kernel": "interp_kernel<double> (S5 weighting pass, fp64)",
            "achieved": rate / 1e9, "peak": peak / 1e9, "unit": "Gpair/s", "frac": rate / peak, "traffic": None,
            "peak_basis": f"{N_SM} SM x {f_max / 1e6:.0f} MHz x {DFMA_PER_CLK_SM} FP64 ops/clk/SM "
                          f"(profiles/r01_pipe_peaks.json) / {DP_ALGO_PER_PAIR} FP64 ops per pair (DESIGN.md §4.9: "
                          f"distance 4, log2 to 2^-36 5, exponent 1, exp2 to 2^-36 8, sums 2)",
            "kernel_fp64_ops_per_pair": DP_PER_PAIR,
            "frac_at_measured_clock": (rate / peak) * (f_max / (clocks["sm_mhz"] * 1e6))
            if clocks.get("sm_mhz") else None}


def fp64_record(per, ms, nq, nq_total, nd, launches, pk):
    f_max = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    pairs = float(nq) * nd
    return {"metric": "AIDW interpolated points/sec (fp64, same workload)", "value": nq_total / (ms / 1e3),
            "unit": "points/s", "ms_per_step": ms, "steps": int(per.shape[0]), "warmup": 3, "dtype": "f64",
            "pair_evals_per_s": 2.0 * nq_total * nd / (ms / 1e3),
            "phases_ms": {"knn_robs": float(per[:, 0].mean()), "allreduce": float(per[:, 1].mean()),
                          "alpha": float(per[:, 2].mean()), "interpolate": float(per[:, 3].mean())},
            "roofline": fp64_roofline(float(per[:, 3].mean()), pairs, f_max, {}),
            "gpu_launches": launches}


if __name__ == "__main__":
    sys.exit(main())
