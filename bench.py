#!/usr/bin/env python
"""bench.py -- throughput of the HP-GWAS hot path on B200 (GLS solves / s), driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--m M] [--impl ours|reference]

A step is one whole job over the rank's synthetic workload:
  gls_create  (potrf of M + inverse, X~_L, y~, S_TL, b_T -- Alg. 5 lines 1,2,4,5,6; on rank 0,
               then one NCCL broadcast of the shared state to the other ranks)
  gls_solve_block over the rank's m SNPs resident in HBM (Alg. 5 line 3 + lines 7-11, fused).
value = SNPs solved by all ranks / max-over-ranks device time (weak scaling: each rank owns a
config-sized SNP range).  e2e = the same through the C ABI with HOST buffers (M, X_L, y and the
rank's X_R in pinned host memory, b back to host) -- the double-buffered H2D stream of Alg. 8.

--impl reference times the CPU oracle (oracle/, the only other place bench.py runs it) on a
bounded sample of the same workload and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gen  # noqa: E402

METRIC = "GLS solves (SNPs)/sec at n=10^4, p=4; FP64 tensor-pipe % of peak, 1/2/4/8 B200"
UNIT = "SNPs/s"
# FP64 tensor (DMMA.8x8x4) peak measured on this pool's B200 by tools/probe (profiles/r01_probe.txt):
# 37.10 TFLOP/s burst, 36.86 TFLOP/s sustained over 4 s.  MEASURED_PEAKS.json carries no FP64 figure.
FP64_DMMA_PEAK_SUSTAINED = 36.86
FP64_DMMA_PEAK_BURST = 37.10
H2D_GBS = 55.6  # pinned host -> device, measured (profiles/r01_probe.txt)
# int8 digit products per FP64 multiply-add of the trsm: T is split into 7 digits
OZ_SLICES = 7


def int8_peak():
    """Dense int8 tensor peak, MEASURED on this pool's B200 by tools/umma_probe/peak_i8.cu
    (profiles/r02_peak_i8.json: tcgen05.mma.cta_group::2.kind::i8, M = 256, N = 224 -- the hot kernel's
    shape -- K = 32, operands resident in shared memory, 148 CTAs).  The hot kernel runs inside a long
    step, so the SUSTAINED figure (back-to-back launches for 4 s) is the denominator; the burst figure
    (one 20 ms launch) is reported beside it.  Fallback when the probe file is absent: 2 x the
    driver-measured bf16 rates of MEASURED_PEAKS.json (nominal int8:bf16 = 4.5:2.25 PF dense).
    Returns (denominator, other, source)."""
    try:
        rows = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r02_peak_i8.json")) if l.strip()]
        r = next(x for x in rows if x.get("N") == 224)
        return (float(r["sustained_tops"]), float(r["burst_tops"]),
                "tcgen05 kind::i8 M=256 N=224 K=32 microbenchmark (tools/umma_probe/peak_i8.cu, "
                "profiles/r02_peak_i8.json): sustained %.1f TOP/s (4 s back to back) is the denominator; "
                "burst %.1f" % (r["sustained_tops"], r["burst_tops"]))
    except Exception:
        pass
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        b, bs = float(mp["bf16_tflops"]), float(mp["bf16_tflops_sustained"])
        return 2.0 * bs, 2.0 * b, ("2 x bf16_tflops_sustained %.1f of MEASURED_PEAKS.json; nominal int8:bf16 = "
                                   "4.5:2.25 PF dense" % bs)
    except Exception:
        return 2.0 * 1400.0, 2.0 * 1590.0, "2 x 1400 TF/s bf16 sustained (B200_PROFILING.md fallback)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--m", "--snps", dest="m", type=int, default=0, help="SNPs per rank (default: the config m)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-records (FP64 path, OOC, weak scaling)")
    ap.add_argument("--scaling", default="auto", choices=["auto", "strong", "weak"],
                    help="auto: strong (the config's m split over the GPUs) when N > 1")
    ap.add_argument("--replicate", default="redundant", choices=["redundant", "bcast", "dist"],
                    help="N > 1: every rank factors M (paper, PAPER.md:812-814), rank 0 + NCCL broadcast, or the "
                         "factorisation split over the ranks (NEXT-3, multi.dist_create)")
    ap.add_argument("--dist-nb", type=int, default=1024, help="column-block width of --replicate dist")
    ap.add_argument("--codes", action="store_true",
                    help="config 4: stream X_R as int8 genotype codes (gls_solve_block_i8) instead of FP64")
    ap.add_argument("--seed", type=int, default=gen.DEFAULT_SEED)
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics only: no nvidia-smi clock sampler "
                    "(a line without it does not meet the timing rules)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region.

    nvidia-smi is launched by `launch()` before the warm-up steps: its start-up (NVML init, first
    query) holds driver locks long enough to stall the host's launches for tens of ms, which showed
    up as 25-77 ms outlier steps when it started with the timed region.  Every row is time-stamped
    on arrival; `start()` / `stop()` bracket the timed region and only rows inside it are kept."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []          # (perf_counter at arrival, fields)
        self._stop = threading.Event()
        self._t = None
        self._t0 = self._t1 = None

    def _run(self):
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                  "--format=csv,noheader,nounits", "-lms", "200"],
                                 stdout=subprocess.PIPE, text=True)
        except Exception:
            return
        while not self._stop.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))
        p.terminate()

    def launch(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def start(self):
        if self._t is None:
            self.launch()
        self._t0 = time.perf_counter()

    def stop(self):
        self._t1 = time.perf_counter()
        # one more sampling interval, so a timed region shorter than it still has a sample
        deadline = self._t1 + 0.5
        while time.perf_counter() < deadline and not any(t >= self._t0 for t, _ in self.rows):
            time.sleep(0.05)
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        inside = [r for t, r in self.rows if self._t0 <= t <= self._t1]
        if not inside:
            inside = [r for t, r in self.rows if t >= self._t0][:1]
        sm = [float(r[0]) for r in inside if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in inside if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in inside:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "sampler": "nvidia-smi -lms 200 launched before the warm-up; rows inside the timed region"}


# ----------------------------------------------------------------------------- oracle arm
def oracle_sample(P, cfg, seed, nsnp, L=None):
    """Time the CPU oracle (as it stands) on `nsnp` seeded SNPs of the workload."""
    import oracle
    t_chol = None
    if L is None:
        t0 = time.perf_counter()
        L = oracle.cholesky(P.M)
        t_chol = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    sel = np.sort(rng.choice(cfg.m, nsnp, replace=False))
    XRs = np.concatenate([gen.make_XR(seed, cfg.n, int(i) * cfg.pR, cfg.pR) for i in sel])
    t0 = time.perf_counter()
    oracle.gls_sequence(L, P.XL, P.y, XRs, cfg.pR, sel=sel, xr_is_selected=True)
    t_snp = time.perf_counter() - t0
    return L, t_chol, t_snp


def cpu_threads():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def workload(args, cfg, world):
    """(scaling, m_total, config dict) of the timed workload -- the same for both arms."""
    scaling = args.scaling if args.scaling != "auto" else ("strong" if world > 1 else "weak")
    m_total = (args.m or cfg.m) * (1 if scaling == "strong" else world)
    conf = {"workload": "config%d: n=%d pL=%d pR=%d, %d SNPs in HBM, %s (rank r owns SNPs [%s))"
                        % (args.config, cfg.n, cfg.pL, cfg.pR, m_total,
                           "split over the GPUs" if scaling == "strong" else "per GPU",
                           "floor(r m/N), floor((r+1) m/N)" if scaling == "strong" else "r m, (r+1) m"),
            "n": cfg.n, "pL": cfg.pL, "pR": cfg.pR, "m_total": m_total, "seed": args.seed}
    return scaling, m_total, conf


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 runs the oracle alone (the other ranks
        # exit at once), so it gets the host's cores -- read by libgomp when oracle/ is first loaded
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    cfg = gen.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    scaling, m, conf = workload(args, cfg, world)
    P = gen.config_problem(cfg, seed=args.seed)
    nsnp = 64 if cfg.n >= 5000 else 512
    L, t_chol, _ = oracle_sample(P, cfg, args.seed, 8)
    times = []
    for s in range(args.warmup + args.steps):
        _, _, t_snp = oracle_sample(P, cfg, args.seed + s, nsnp, L=L)
        if s >= args.warmup:
            times.append(t_snp)
    rate = nsnp / statistics.median(times)
    value = m / (t_chol + m / rate)
    sample = ("oracle Cholesky of the full n=%d M (%.2f s, once) + %d seeded SNPs per step (Alg. 4 "
              "per-problem steps); value = m / (t_chol + m / rate), m = the whole job's %d SNPs"
              % (cfg.n, t_chol, nsnp, m))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": conf,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
class Job:
    """One rank's share of a config-2-shaped workload resident in HBM, and the step that solves it:
    gls_create (each rank factors M itself -- the paper's "factorization of M redundantly",
    PAPER.md:812-814 -- or rank 0 factors and broadcasts, --replicate bcast) + gls_solve_block over
    the rank's SNPs, on a dedicated stream whose CUDA events bracket the library's launches."""

    def __init__(self, args, cfg, P, world, rank, m_rank, g0, torch, pkg, multi, dist):
        self.args, self.cfg, self.P, self.world, self.rank = args, cfg, P, world, rank
        self.m, self.g0 = m_rank, g0
        self.torch, self.pkg, self.multi, self.dist = torch, pkg, multi, dist
        n, pR, p = cfg.n, cfg.pR, cfg.p
        self.Md = torch.from_numpy(P.M).cuda()
        self.XLd = torch.from_numpy(np.ascontiguousarray(P.XL)).cuda()
        self.yd = torch.from_numpy(P.y).cuda()
        self.Xd = torch.empty((max(m_rank, 1) * pR, n), dtype=torch.float64, device="cuda")
        chunk = 65536
        for c in range(0, m_rank * pR, chunk):
            k = min(chunk, m_rank * pR - c)
            pkg.gen_xr_device(args.seed, n, g0 * pR + c, k, self.Xd[c:c + k])
        self.b = torch.empty((max(m_rank, 1), p), dtype=torch.float64, device="cuda")
        self.st = torch.empty(max(m_rank, 1), dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        # a real (non-legacy) stream: the library's kernels are enqueued on it via gls_set_stream,
        # so CUDA events recorded on it bracket exactly the fused kernel
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)

    def make_ctx(self, Mx, XLx, yx, async_create=False):
        cfg, pkg = self.cfg, self.pkg
        if self.args.replicate == "dist":
            # NEXT-3: the factorisation itself split over the ranks (column blocks of M and T, panel
            # broadcasts); every rank ends with the same int8-only state
            return self.multi.dist_create(cfg.n, cfg.pL, cfg.pR, Mx, XLx, yx, dist=self.dist if self.world > 1 else None,
                                          nb=self.args.dist_nb)
        if self.world > 1 and self.args.replicate == "bcast":
            ctx = (pkg.Context(cfg.n, cfg.pL, cfg.pR, Mx, XLx, yx) if self.rank == 0
                   else pkg.Context(cfg.n, cfg.pL, cfg.pR, adopt=True))
            self.multi.replicate_shared(ctx, self.dist, src=0)
        else:
            ctx = pkg.Context(cfg.n, cfg.pL, cfg.pR, Mx, XLx, yx, async_create=async_create)
        return ctx

    def run(self, steps, warmup, path=None, clocks=None):
        torch, dist, multi = self.torch, self.dist, self.multi
        kern_ms, create_ms, timing, launches = [], [], [], [0]

        hostlog = os.environ.get("GLS_BENCH_HOSTLOG") == "1"   # diagnostics: host time of each call

        def step(timed):
            tc = time.perf_counter()
            ctx = self.make_ctx(self.Md, self.XLd, self.yd)
            th = [tc, time.perf_counter()]
            if timed:
                create_ms.append(1e3 * (th[1] - tc))
            if path is not None:
                ctx.set_path(path)
            ctx.set_stream(self.stream.cuda_stream)
            ctx.set_timing(timed)
            k0 = torch.cuda.Event(enable_timing=True)
            k1 = torch.cuda.Event(enable_timing=True)
            k0.record(self.stream)
            th.append(time.perf_counter())
            if self.m > 0:
                ctx.solve_block(self.Xd, self.m, self.b, self.st, async_=True)
            k1.record(self.stream)
            th.append(time.perf_counter())
            ctx.sync()
            th.append(time.perf_counter())
            if timed:
                launches[0] += ctx.kernel_launches
                k1.synchronize()
                kern_ms.append(k0.elapsed_time(k1))
                timing.append(ctx.read_timing())
                timing[-1]["paths"] = ctx.path_counts()
            th.append(time.perf_counter())
            ctx.close()
            th.append(time.perf_counter())
            if hostlog:
                names = ("create", "setup", "enqueue", "sync", "read", "close")
                print("[host] " + " ".join("%s %.2f" % (nm, 1e3 * (th[i + 1] - th[i])) for i, nm in enumerate(names)),
                      file=sys.stderr, flush=True)

        if clocks:
            clocks.launch()     # nvidia-smi's start-up lands in the warm-up, not in a timed step
        for _ in range(warmup):
            step(False)
        if clocks:
            clocks.start()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        marks = []
        for _ in range(steps):
            step(True)
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record(self.stream)
        e1.record(self.stream)
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        clk = clocks.stop() if clocks else None
        total_ms = e0.elapsed_time(e1)
        each = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i]) for i in range(1, len(marks))]
        vals = multi.max_over_ranks([total_ms, statistics.mean(kern_ms),
                                     statistics.mean(t["int8_ms"] for t in timing),
                                     statistics.mean(t["fp64_ms"] for t in timing),
                                     statistics.mean(t["conv_ms"] for t in timing),
                                     statistics.mean(create_ms)], dist, device="cuda")
        return {"ms_per_step": vals[0] / steps, "solve_block_ms": vals[1], "int8_ms": vals[2], "fp64_ms": vals[3],
                "conv_ms": vals[4], "create_ms": vals[5], "paths": timing[-1]["paths"], "launches": launches[0],
                "step_ms_rank": [round(x, 2) for x in each], "create_ms_rank": [round(x, 2) for x in create_ms],
                "solve_ms_rank": [round(x, 2) for x in kern_ms],
                "clocks": clk}


def int8_roofline(r, n, m, pR, traffic):
    flops = float(n) * n * m * pR          # FP64 trsm flops, n^2 per X_R column (north star)
    ops = OZ_SLICES * flops                # int8 ops: 7 digit products per FP64 MAC
    peak, peak_burst, psrc = int8_peak()
    achieved = ops / (r["int8_ms"] / 1e3) / 1e12
    fp64eq = flops / (r["int8_ms"] / 1e3) / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
            "frac": achieved / peak, "traffic": traffic, "kernel": "ozaki_trsm_gls_kernel",
            "kernel_ms": r["int8_ms"],
            "kernel_includes": "the FP64 -> int8 conversion of the next chunk's X_R (two convert-ahead "
                               "warps, concurrent with the MMAs; only the first chunk's pass is separate)",
            "fp64_fallback_ms": r["fp64_ms"] if r["paths"][1] > 0 else 0.0,
            "solve_block_ms": r["solve_block_ms"], "exposed_overhead_ms": r["solve_block_ms"] - r["int8_ms"],
            "create_ms": r["create_ms"], "int8_ops_per_launch": ops, "peak_source": psrc,
            "frac_of_burst_peak": achieved / peak_burst, "burst_peak": peak_burst,
            "fp64_equivalent": {"achieved_tflops": fp64eq, "dmma_peak_tflops": FP64_DMMA_PEAK_SUSTAINED,
                                "ratio_to_dmma_peak": fp64eq / FP64_DMMA_PEAK_SUSTAINED,
                                "note": "n^2 FP64 trsm flops per column / kernel time; the FP64 DMMA pipe "
                                        "peak is measured in profiles/r01_probe.txt"}}


def fp64_roofline(r, n, m, pR, traffic):
    flops = float(n) * n * m * pR
    achieved = flops / (r["fp64_ms"] / 1e3) / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": FP64_DMMA_PEAK_SUSTAINED, "unit": "TFLOP/s",
            "frac": achieved / FP64_DMMA_PEAK_SUSTAINED, "traffic": traffic, "kernel": "fused_trsm_gls_kernel",
            "kernel_ms": r["fp64_ms"], "solve_block_ms": r["solve_block_ms"], "create_ms": r["create_ms"],
            "flops_per_launch": flops,
            "peak_source": "FP64 DMMA.8x8x4 microbenchmark on this pool's B200, 4 s sustained "
                           "(profiles/r01_probe.txt); MEASURED_PEAKS.json has no FP64 entry"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1210_7325_b200 as pkg
    from paper_1210_7325_b200 import multi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # GLS_BENCH_DEVICE / GLS_BENCH_BACKEND: functional checks of the N > 1 code path with several ranks
    # on one GPU over gloo (tools/sessions/gpu_run13.sh); never used for a measurement
    local = int(os.environ.get("GLS_BENCH_DEVICE", multi.local_device()))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("GLS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    pkg.load()
    # No cyclic-GC pauses inside timed regions: after torch's imports a full collection walks ~170k
    # objects (~75 ms), and one landing in a step stalls the host between that step's synchronising
    # calls -- seen as single 55-93 ms outlier steps (create or close).  Collect once here, then off.
    gc.collect()
    if os.environ.get("GLS_BENCH_GC") != "1":   # diagnostics: keep the collector on
        gc.disable()

    cfg = gen.CONFIGS[args.config]
    if args.config == 4:
        return run_ooc(args, cfg, world, rank, local)
    n, pL, pR, p = cfg.n, cfg.pL, cfg.pR, cfg.p
    scaling, m_total, conf = workload(args, cfg, world)
    if scaling == "strong":
        g0, g1 = multi.snp_range(m_total, world, rank)   # the config's m split over the ranks
    else:
        g0, g1 = multi.weak_range(args.m or cfg.m, rank)  # every rank owns a config-sized range
    m = g1 - g0
    P = gen.config_problem(cfg, seed=args.seed)
    job = Job(args, cfg, P, world, rank, m, g0, torch, pkg, multi, dist)

    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("config%d" % args.config)
        except Exception:
            traffic = None

    r = job.run(args.steps, args.warmup, clocks=None if args.no_clocks else ClockSampler(local))
    value = m_total / (r["ms_per_step"] / 1e3)
    n_bad = int(job.st[:m].sum().item()) if m else 0
    b_ref = job.b[:m].cpu()  # the main run's b (the sub-records below reuse job.b)
    m_max = max(multi.max_over_ranks([float(m)], dist, device="cuda"))
    roofline = (int8_roofline(r, n, int(m_max), pR, traffic) if r["paths"][0] > 0
                else fp64_roofline(r, n, int(m_max), pR, traffic))
    solve_only = m_total / (r["solve_block_ms"] / 1e3)

    # ---- evidence that every rank holds the same shared state (redundant factorisations)
    replication = None
    if world > 1:
        ctx = job.make_ctx(job.Md, job.XLd, job.yd)
        dg = torch.tensor(multi.shared_state_digest(ctx), dtype=torch.int64, device="cuda")
        ctx.close()
        hi, lo = dg.clone(), dg.clone()
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        replication = {"mode": args.replicate, "shared_state_bitwise_equal_across_ranks": bool(torch.equal(hi, lo)),
                       "evidence": "per-buffer 64-bit digests of the shared state (multi.shared_state_digest), "
                                   "min == max over ranks"}

    # ---- sub-records (fixed small step counts, so the default run stays within minutes)
    subs = {}
    if not args.no_sub and r["paths"][0] > 0 and args.replicate != "dist":
        # the FP64 tensor-pipe path on the same workload: the metric's "FP64 tensor-pipe % of peak"
        r64 = job.run(2, 1, path=pkg.GLS_PATH_FP64)
        rl64 = fp64_roofline(r64, n, int(m_max), pR, None)
        subs["fp64_path"] = {"value": m_total / (r64["ms_per_step"] / 1e3), "unit": UNIT, "steps": 2, "warmup": 1,
                             "ms_per_step": r64["ms_per_step"],
                             "fp64_tensor_pipe_pct_of_peak": 100.0 * rl64["frac"], "roofline": rl64,
                             "arithmetic": "FP64 on the DMMA tensor pipe (GLS_PATH_FP64), same step, same data"}
    # ---- e2e: the same job through the C ABI with HOST buffers, host<->device copies inside the
    # timed region (Alg. 8 double-buffered stream).  Primary: X_R as genotype codes (int8, one byte
    # per genotype -- gls_solve_block_i8); secondary: X_R as FP64 (gls_solve_block, 8 bytes).
    e2e = None
    if not args.no_e2e and job.m > 0:
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except (ValueError, OSError):
            avail = 1 << 40
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        Mh = torch.from_numpy(P.M).pin_memory()
        XLh = torch.from_numpy(np.ascontiguousarray(P.XL)).pin_memory()
        yh = torch.from_numpy(P.y).pin_memory()
        mj = job.m

        def timed_e2e(solve, m_e, steps):
            bh = torch.empty((m_e, p), dtype=torch.float64, pin_memory=True)
            sh = torch.empty(m_e, dtype=torch.int32, pin_memory=True)

            def one():
                # gls_create_async: the first X_R chunks stream in while M is factored (the paper's
                # first block load, otherwise exposed -- PAPER.md:723-728); the synchronous solve
                # below resolves the create's outcome
                ctx = job.make_ctx(Mh, XLh, yh, async_create=True)
                ctx.set_stream_report(True)
                solve(ctx, m_e, bh, sh)
                rep = ctx.read_stream_report()
                ctx.close()
                return rep

            for _ in range(max(1, min(args.warmup, 3))):   # the first steps still page in pinned buffers
                one()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = [one() for _ in range(steps)]
            torch.cuda.synchronize()
            dt = multi.max_over_ranks([(time.perf_counter() - t0) / steps], dist, device="cuda")[0]
            return dt, bool(torch.equal(bh, b_ref[:m_e])), overlap_summary(reps[-1])

        chunk = 65536
        m_i8 = int(min(mj, 0.6 * avail / local_world / (n * pR)))
        m_i8 = max(m_i8 - m_i8 % 64, 64) if m_i8 < mj else mj
        Gh = torch.empty((m_i8 * pR, n), dtype=torch.int8, pin_memory=True)
        for c in range(0, m_i8 * pR, chunk):
            k = min(chunk, m_i8 * pR - c)
            Gh[c:c + k].copy_(job.Xd[c:c + k].to(torch.int8))
        dt8, same8, ov8 = timed_e2e(lambda ctx, me, bh, sh: ctx.solve_block_i8(Gh, me, bh, sh), m_i8, args.steps)
        del Gh
        m_i8_all = multi.sum_over_ranks([float(m_i8)], dist, device="cuda")[0]
        e2e = {"value": m_i8_all / dt8, "unit": UNIT,
               "h2d_bytes_per_step": int((n * n + n * (pL + 1)) * 8 + m_i8 * pR * n),
               "d2h_bytes_per_step": int(m_i8 * p * 8 + m_i8 * 4),
               "m_per_rank": m_i8, "overlap": ov8,
               "path": "C ABI gls_create_async + gls_solve_block_i8: M, X_L, y (FP64) and X_R as int8 "
                       "genotype codes in pinned host memory -> double-buffered H2D stream, its first chunks "
                       "copied while M is factored; b and status back to pinned host memory",
               "bitwise_equal_to_device_run": same8}
        # FP64 X_R from host (8 bytes per genotype over PCIe): a SUBSET of the rank's SNPs (at most 250k,
        # 20 GB of pinned memory per rank at n = 1e4), 2 timed steps
        m_f = int(min(mj, 250_000, 0.6 * avail / local_world / (n * pR * 8)))
        m_f = max(m_f - m_f % 64, 64)
        Xh = torch.empty((m_f * pR, n), dtype=torch.float64, pin_memory=True)
        for c in range(0, m_f * pR, chunk):
            k = min(chunk, m_f * pR - c)
            Xh[c:c + k].copy_(job.Xd[c:c + k])
        dtf, samef, ovf = timed_e2e(lambda ctx, me, bh, sh: ctx.solve_block(Xh, me, bh, sh), m_f, 2)
        del Xh
        m_f_all = multi.sum_over_ranks([float(m_f)], dist, device="cuda")[0]
        e2e["fp64_host_input"] = {"value": m_f_all / dtf, "unit": UNIT, "m_per_rank": m_f,
                                  "subset": m_f < mj,
                                  "note": "a subset of the rank's SNPs (PCIe-bound: 8 bytes per genotype); "
                                          "rate = subset SNPs / subset time",
                                  "h2d_bytes_per_step": int((n * n + n * (pL + 1) + m_f * pR * n) * 8),
                                  "d2h_bytes_per_step": int(m_f * p * 8 + m_f * 4), "overlap": ovf,
                                  "h2d_roofline_snps_per_s": H2D_GBS * 1e9 / (8.0 * n * pR),
                                  "path": "C ABI gls_create_async + gls_solve_block, FP64 X_R in pinned host memory",
                                  "bitwise_equal_to_device_run": samef}

    if world > 1 and scaling == "strong" and not args.no_sub:
        # weak scaling as a labelled sub-record: every rank owns a full config-sized range
        job = None
        torch.cuda.empty_cache()
        mw = args.m or cfg.m
        gw0, gw1 = multi.weak_range(mw, rank)
        jw = Job(args, cfg, P, world, rank, mw, gw0, torch, pkg, multi, dist)
        rw = jw.run(2, 1)
        subs["weak_scaling"] = {"value": world * mw / (rw["ms_per_step"] / 1e3), "unit": UNIT,
                                "m_per_rank": mw, "ms_per_step": rw["ms_per_step"], "steps": 2, "warmup": 1}
        del jw

    # ---- config-3 shape (p = 20) and file out-of-core (NEXT-1) sub-records: driver-observed evidence
    if not args.no_sub and args.config == 2 and world == 1:
        job = None
        torch.cuda.empty_cache()
        subs["config3_reduced"] = config3_subrecord(args, world, rank, pkg, multi, dist, torch)
        torch.cuda.empty_cache()
        try:
            subs["file_ooc_next1"] = file_ooc_subrecord(args, pkg, torch)
        except Exception as e:  # a box without a writable local disk: say so, keep the line
            subs["file_ooc_next1"] = {"unavailable": str(e)[:200]}

    # ---- out-of-core sub-record (config-4 shape, reduced m): the Alg. 8 stream from pinned host
    # memory, codes and FP64, with the overlap accounting of every chunk
    if not args.no_sub and args.config == 2:
        job = None
        torch.cuda.empty_cache()
        subs["ooc_config4_reduced"] = ooc_subrecord(args, gen.CONFIGS[4], world, rank, pkg, multi, dist, torch)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nsnp = 64 if n >= 5000 else 512
        L, t_chol, t_snp = oracle_sample(P, cfg, args.seed, nsnp)
        rate = nsnp / t_snp
        cpu = {"value": m_total / (t_chol + m_total / rate), "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
               "sample": "oracle Cholesky of the full n=%d M (%.2f s) + %d seeded SNPs of the workload "
                         "(%.2f s); value = m / (t_chol + m / rate)" % (n, t_chol, nsnp, t_snp)}

    if rank == 0:
        int8 = roofline["kernel"].startswith("ozaki")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None,
                "dtype": "f64 (exact int8x7 digit products)" if int8 else "f64",
                "data": "synthetic",
                "arithmetic": ("FP64 results; the trsm as exact int8 x int8 -> int32 digit products on tcgen05 "
                               "(T = L^-1 split into 7 base-256 digits, 55 bits per row; X_R integer) combined "
                               "and reduced in FP64 (DESIGN.md reading A15)") if int8
                              else "FP64 on the DMMA tensor pipe",
                "config": {**conf, "m_per_rank_max": int(m_max), "replicate": args.replicate if world > 1 else None,
                           "step": "gls_create (every rank factors M itself, or rank 0 + NCCL broadcast) + "
                                   "gls_solve_block over the rank's SNPs",
                           "l2": "inputs larger than L2 (X_R %.1f GB per rank)" % (m_max * pR * n * 8 / 1e9)},
                "solve_only": {"value": solve_only, "unit": UNIT,
                               "note": "SNPs / gls_solve_block time, gls_create excluded (SURVEY §8(d)'s timed "
                                       "region); value above includes gls_create every step"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": r["launches"],
                "clocks": r["clocks"], "step_ms_rank0": r["step_ms_rank"], "create_ms_rank0": r["create_ms_rank"],
                "solve_ms_rank0": r["solve_ms_rank"],
                "rank_deficient_rows": n_bad, "replication": replication, **subs}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def overlap_summary(rep):
    """Fractions of the stream report (gls_read_stream_report) for the JSON line."""
    w = rep["wall_ms"] or 1e-9
    exposed = rep["first_load_ms"] + rep["exposed_h2d_ms"] + rep["exposed_other_ms"] + rep["tail_ms"]
    return {"chunks": rep["chunks"], "wall_ms": rep["wall_ms"], "h2d_busy_frac": rep["h2d_ms"] / w,
            "compute_busy_frac": rep["compute_ms"] / w, "d2h_busy_frac": rep["d2h_ms"] / w,
            "exposed_wait_pct": 100.0 * exposed / w, "first_load_ms": rep["first_load_ms"],
            "exposed_h2d_ms": rep["exposed_h2d_ms"], "exposed_other_ms": rep["exposed_other_ms"],
            "tail_ms": rep["tail_ms"], "h2d_gbs": rep["h2d_bytes"] / max(rep["h2d_ms"], 1e-9) / 1e6}


def config3_subrecord(args, world, rank, pkg, multi, dist, torch):
    """Config 3's shape (n = 1e4, pL = 16 covariates, pR = 4: p = 20) with a reduced m of 1e5 groups
    (32 GB of X_R in HBM): the same step (create + solve), 1 warm-up and 2 timed steps, int8 roofline."""
    cfg = gen.CONFIGS[3]
    mg = 100_000
    P = gen.config_problem(cfg, seed=args.seed)
    a2 = argparse.Namespace(**vars(args))
    a2.replicate = "redundant"
    j = Job(a2, cfg, P, world, rank, mg, 0, torch, pkg, multi, dist)
    r = j.run(2, 1)
    rl = int8_roofline(r, cfg.n, mg, cfg.pR, None)
    return {"value": mg / (r["ms_per_step"] / 1e3), "unit": "GLS solves (SNP groups of pR = 4)/s",
            "m_groups": mg, "n": cfg.n, "pL": cfg.pL, "pR": cfg.pR, "ms_per_step": r["ms_per_step"],
            "steps": 2, "warmup": 1, "create_ms": r["create_ms"], "int8_kernel_ms": r["int8_ms"],
            "roofline_frac": rl["frac"], "achieved_int8_tops": rl["achieved"], "paths": r["paths"]}


def file_ooc_subrecord(args, pkg, torch):
    """NEXT-1 (§4): 1e6 config-4 SNPs as int8 genotype codes (10 GB) in a file on the box's local disk,
    solved with gls_solve_file in Alg. 7 (synchronous) and Alg. 8 (double-buffered) mode, each from a
    cold page cache; the raw O_DIRECT read rate of the same file is the I/O roofline."""
    import mmap
    import tempfile
    cfg = gen.CONFIGS[4]
    n, pL, pR, m = cfg.n, cfg.pL, cfg.pR, 1_000_000
    P = gen.config_problem(cfg, seed=args.seed)
    d = tempfile.mkdtemp(prefix="gls_ooc_", dir=os.environ.get("GLS_OOC_DIR", "/tmp"))
    xr, bf = os.path.join(d, "xr_i8.bin"), os.path.join(d, "b.bin")

    def evict(path):
        fd = os.open(path, os.O_RDONLY)
        os.fsync(fd)
        os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
        os.close(fd)

    try:
        tmp = torch.empty((65536, n), dtype=torch.float64, device="cuda")
        with open(xr, "wb") as f:
            for c in range(0, m, 65536):
                k = min(65536, m - c)
                pkg.gen_xr_device(args.seed, n, c, k, tmp[:k])
                f.write(tmp[:k].to(torch.int8).cpu().numpy().tobytes())
        del tmp
        size = os.path.getsize(xr)
        evict(xr)
        buf = mmap.mmap(-1, 512 << 20)  # large O_DIRECT requests, as the engine's 758 MB block reads
        t0 = time.perf_counter()
        fd = os.open(xr, os.O_RDONLY | getattr(os, "O_DIRECT", 0))
        off = 0
        while True:
            got = os.preadv(fd, [buf], off)
            if got <= 0:
                break
            off += got
        os.close(fd)
        read_gbs = size / (time.perf_counter() - t0) / 1e9
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        out = {"m": m, "file_bytes": size, "raw_read_gbs": read_gbs, "block_snps": 148 * 128 * 4,
               "warmup_block_snps": 148 * 128}
        bits = []
        with pkg.Context(n, pL, pR, dv(P.M), dv(P.XL), dv(P.y)) as ctx:
            for name, mode in (("alg7_sync", pkg.GLS_OOC_SYNC), ("alg8_double_buffered", pkg.GLS_OOC_ASYNC)):
                evict(xr)
                rep = ctx.solve_file(xr, m, bf, elem_bytes=1, block_groups=148 * 128 * 4,
                                     warmup_groups=148 * 128, mode=mode)
                bits.append(open(bf, "rb").read())
                rep["snps_per_s"] = m / rep["wall_s"]
                rep["io_roofline_frac"] = (size / (read_gbs * 1e9)) / rep["wall_s"]
                out[name] = rep
        out["alg7_over_alg8"] = out["alg7_sync"]["wall_s"] / out["alg8_double_buffered"]["wall_s"]
        out["bitwise_equal"] = bits[0] == bits[1]
        return out
    finally:
        for f in (xr, bf):
            if os.path.exists(f):
                os.remove(f)
        os.rmdir(d)


def ooc_subrecord(args, cfg, world, rank, pkg, multi, dist, torch):
    """Config-4-shaped out-of-core stream with a reduced m (2e6 SNPs per rank): the blocks of a pool
    of 2 distinct pinned host blocks cycled (block j = pool block j mod 2), once as int8 genotype codes
    and once as FP64, one warm-up and one timed pass each, with per-chunk overlap accounting."""
    from paper_1210_7325_b200 import ooc
    n, pL, pR, p = cfg.n, cfg.pL, cfg.pR, cfg.p
    m = 2_000_000
    P = gen.config_problem(cfg, seed=args.seed)
    Md = torch.from_numpy(P.M).cuda()
    XLd = torch.from_numpy(np.ascontiguousarray(P.XL)).cuda()
    yd = torch.from_numpy(P.y).cuda()
    blk = ooc.host_block_groups(torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count, pR)
    g0 = multi.weak_range(m, rank)[0]
    # pinned pool per rank: 2 blocks (FP64 + codes: ~13.6 GB at n = 1e4), or 1 when the host is short
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 1 << 40
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    npool = 2 if 2 * blk * pR * n * 9 <= 0.4 * avail / local_world else 1
    tmp = torch.empty((blk * pR, n), dtype=torch.float64, device="cuda")
    pool64 = torch.empty((npool, blk * pR, n), dtype=torch.float64, pin_memory=True)
    pool8 = torch.empty((npool, blk * pR, n), dtype=torch.int8, pin_memory=True)
    for k in range(npool):
        pkg.gen_xr_device(args.seed, n, (g0 + k * blk) * pR, blk * pR, tmp)
        pool64[k].copy_(tmp)
        pool8[k].copy_(tmp.to(torch.int8))
    del tmp
    b = torch.empty((m, p), dtype=torch.float64, pin_memory=True)
    st = torch.empty(m, dtype=torch.int32, pin_memory=True)
    out = {"m_per_rank": m, "block_snps": blk, "pool_blocks": npool,
           "snp_to_block": "block j -> pool block j mod %d" % npool, "steps": 1, "warmup": 1}
    peak8, _, _ = int8_peak()
    for name, pool, codes, esz in (("codes", pool8, True, 1), ("fp64", pool64, False, 8)):
        res = None
        for it in range(2):
            ctx = pkg.Context(n, pL, pR, Md, XLd, yd)
            ctx.set_stream_report(True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ooc.stream_from_pool(ctx, pool, m, blk, b, st, codes=codes)
            dt = time.perf_counter() - t0
            rep = ctx.read_stream_report()
            ctx.close()
            res = (dt, rep)
        dt, rep = res
        dt = multi.max_over_ranks([dt], dist, device="cuda")[0]
        t_comp = OZ_SLICES * float(n) * n * m * pR / (peak8 * 1e12)
        t_h2d = float(esz) * n * m * pR / (H2D_GBS * 1e9)
        out[name] = {"value": world * m / dt, "unit": UNIT, "s_per_pass": dt,
                     "bound": "tensor (int8)" if t_comp >= t_h2d else "h2d",
                     "roofline_frac": max(t_comp, t_h2d) / dt,
                     "t_compute_roofline_s": t_comp, "t_h2d_roofline_s": t_h2d,
                     "h2d_bytes": int(esz * n * m * pR), "overlap": overlap_summary(rep)}
    return out


# ----------------------------------------------------------------------------- config 4 (OOC)
def run_ooc(args, cfg, world, rank, local):
    """Config 4: m = 1e7 SNPs per rank streamed from pinned host memory through the double-buffered
    H2D pipeline of gls_solve_block (Alg. 8).  800 GB does not fit in host RAM,
    so a pool of distinct pinned blocks (as much as 50 % of free RAM allows) is cycled: chunk j of
    the rank's stream is pool block j mod P (the SNP -> block map is recorded in the JSON line).
    Every byte still crosses PCIe, so the H2D roofline is unchanged."""
    import torch
    import torch.distributed as dist

    import paper_1210_7325_b200 as pkg
    from paper_1210_7325_b200 import multi

    n, pL, pR, p = cfg.n, cfg.pL, cfg.pR, cfg.p
    m = args.m or cfg.m
    P = gen.config_problem(cfg, seed=args.seed)
    Md = torch.from_numpy(P.M).cuda()
    XLd = torch.from_numpy(np.ascontiguousarray(P.XL)).cuda()
    yd = torch.from_numpy(P.y).cuda()
    from paper_1210_7325_b200 import ooc
    props = torch.cuda.get_device_properties(local)
    # block = the library's default host chunk: 4 waves of 128-column int8 tiles
    blk_groups = ooc.host_block_groups(props.multi_processor_count, pR)
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 1 << 40
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    esz = 1 if args.codes else 8
    blk_bytes = blk_groups * pR * n * esz
    nblk = (m + blk_groups - 1) // blk_groups
    pool_n = int(max(2, min(nblk, 0.5 * avail / local_world // blk_bytes)))
    g0 = multi.weak_range(m, rank)[0]
    pool = torch.empty((pool_n, blk_groups * pR, n), dtype=torch.int8 if args.codes else torch.float64,
                       pin_memory=True)
    tmp = torch.empty((blk_groups * pR, n), dtype=torch.float64, device="cuda")
    for k in range(pool_n):
        pkg.gen_xr_device(args.seed, n, (g0 + k * blk_groups) * pR, blk_groups * pR, tmp)
        pool[k].copy_(tmp.to(torch.int8) if args.codes else tmp)
    del tmp
    b = torch.empty((m, p), dtype=torch.float64, pin_memory=True)
    st = torch.empty(m, dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()

    def step():
        ctx = pkg.Context(n, pL, pR, Md, XLd, yd) if rank == 0 else pkg.Context(n, pL, pR, adopt=True)
        if world > 1:
            multi.replicate_shared(ctx, dist, src=0)
        ooc.stream_from_pool(ctx, pool, m, blk_groups, b, st, codes=args.codes)
        launches = ctx.kernel_launches
        ctx.close()
        return launches

    clocks = ClockSampler(local)
    clocks.launch()
    for _ in range(max(1, args.warmup)):
        step()
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    launches = 0
    for _ in range(args.steps):
        launches += step()
    torch.cuda.synchronize()
    dt = multi.max_over_ranks([(time.perf_counter() - t0) / args.steps], dist, device="cuda")[0]
    clk = clocks.stop()
    value = world * m / dt
    # int8 path (genotypes): 7 n^2 int8 ops per column at the int8 peak; H2D: esz bytes per genotype
    peak8, _, psrc = int8_peak()
    t_comp = OZ_SLICES * float(n) * n * m * pR / (peak8 * 1e12)
    t_h2d = float(esz) * n * m * pR / (H2D_GBS * 1e9)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * dt, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "config4: n=%d pL=%d pR=%d, %d SNPs per GPU streamed from pinned "
                                       "host memory in %d-SNP chunks (out-of-core, Alg. 8), X_R as %s"
                                       % (n, pL, pR, m, blk_groups,
                                          "int8 genotype codes" if args.codes else "FP64"),
                           "n": n, "m_per_rank": m, "chunk_snps": blk_groups,
                           "host_pool_blocks": pool_n, "snp_to_block": "chunk j -> pool block j mod %d" % pool_n,
                           "l2": "inputs larger than L2"},
                "roofline": {"bound": "tensor" if t_comp >= t_h2d else "h2d",
                             "achieved": (OZ_SLICES * float(n) * n * m * pR / dt / 1e12) if t_comp >= t_h2d
                             else float(esz) * n * m * pR / dt / 1e9,
                             "peak": peak8 if t_comp >= t_h2d else H2D_GBS,
                             "unit": "TOP/s (int8)" if t_comp >= t_h2d else "GB/s (H2D)",
                             "frac": max(t_comp, t_h2d) / dt, "traffic": None,
                             "t_compute_roofline_s": t_comp, "t_h2d_roofline_s": t_h2d,
                             "h2d_gbs_measured": H2D_GBS, "int8_peak_source": psrc},
                "cpu_baseline": None,
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(esz * n * m * pR + 8 * n * n),
                        "d2h_bytes_per_step": int(m * p * 8 + m * 4),
                        "path": "C ABI, host X_R -> double-buffered H2D (the whole step is end to end)"},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
