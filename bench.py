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
    """Dense int8 tensor peak: the driver-measured bf16 GEMM rate (MEASURED_PEAKS.json) x the nominal
    int8:bf16 ratio 4.5:2.25 (B200_PROFILING.md).  The BURST figure is the denominator: the kernel
    runs inside a long step, but it measurably exceeds 2 x the sustained bf16 rate (it draws less
    power than a dense bf16 GEMM), so the sustained figure would not bound it."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        b, bs = float(mp["bf16_tflops"]), float(mp["bf16_tflops_sustained"])
        return 2.0 * b, 2.0 * bs, ("2 x bf16_tflops %.1f (burst) of MEASURED_PEAKS.json; nominal int8:bf16 = "
                                   "4.5:2.25 PF dense" % b)
    except Exception:
        return 2.0 * 1590.0, 2.0 * 1400.0, "2 x 1590 TF/s bf16 burst (B200_PROFILING.md fallback)"


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
    ap.add_argument("--codes", action="store_true",
                    help="config 4: stream X_R as int8 genotype codes (gls_solve_block_i8) instead of FP64")
    ap.add_argument("--seed", type=int, default=gen.DEFAULT_SEED)
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

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
            self.rows.append([x.strip() for x in line.split(",")])
        p.terminate()

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


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


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = gen.CONFIGS[args.config]
    m = args.m or cfg.m
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
              "per-problem steps); value = m / (t_chol + m / rate)" % (cfg.n, t_chol, nsnp))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "config%d" % args.config, "n": cfg.n, "pL": cfg.pL, "pR": cfg.pR,
                       "m_per_rank": m},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
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
    local = multi.local_device()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    pkg.load()

    cfg = gen.CONFIGS[args.config]
    if args.config == 4:
        return run_ooc(args, cfg, world, rank, local)
    n, pL, pR, p = cfg.n, cfg.pL, cfg.pR, cfg.p
    m = args.m or cfg.m
    col0 = multi.weak_range(m, rank)[0] * pR  # this rank's SNP range [rank*m, (rank+1)*m)

    P = gen.config_problem(cfg, seed=args.seed)
    Md = torch.from_numpy(P.M).cuda()
    XLd = torch.from_numpy(np.ascontiguousarray(P.XL)).cuda()
    yd = torch.from_numpy(P.y).cuda()
    Xd = torch.empty((m * pR, n), dtype=torch.float64, device="cuda")
    chunk = 65536
    for c in range(0, m * pR, chunk):
        k = min(chunk, m * pR - c)
        pkg.gen_xr_device(args.seed, n, col0 + c, k, Xd[c:c + k])
    b = torch.empty((m, p), dtype=torch.float64, device="cuda")
    st = torch.empty(m, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    # a real (non-legacy) stream: the library's kernels are enqueued on it via gls_set_stream,
    # so CUDA events recorded on it bracket exactly the fused kernel
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def make_ctx(Mx, XLx, yx):
        # rank 0 factors; the others adopt the broadcast shared state
        if rank == 0:
            ctx = pkg.Context(n, pL, pR, Mx, XLx, yx)
        else:
            ctx = pkg.Context(n, pL, pR, adopt=True)
        if world > 1:
            multi.replicate_shared(ctx, dist, src=0)
        return ctx

    kern_ms = []
    create_ms = []
    timing = []
    launches = [0]

    def step(timed: bool):
        tc = time.perf_counter()
        ctx = make_ctx(Md, XLd, yd)
        if timed:
            create_ms.append(1e3 * (time.perf_counter() - tc))
        ctx.set_stream(stream.cuda_stream)
        ctx.set_timing(timed)
        k0 = torch.cuda.Event(enable_timing=True)
        k1 = torch.cuda.Event(enable_timing=True)
        k0.record(stream)
        ctx.solve_block(Xd, m, b, st, async_=True)
        k1.record(stream)
        ctx.sync()
        if timed:
            launches[0] += ctx.kernel_launches
            k1.synchronize()
            kern_ms.append(k0.elapsed_time(k1))
            timing.append(ctx.read_timing())
            timing[-1]["paths"] = ctx.path_counts()
        ctx.close()

    for _ in range(args.warmup):
        step(False)
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(True)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    total_ms, kern_avg_ms = multi.max_over_ranks([total_ms, statistics.mean(kern_ms)], dist, device="cuda")
    ms_per_step = total_ms / args.steps
    value = world * m / (ms_per_step / 1e3)

    # parity spot check of this run's output against the planted structure is in tests/; here only
    # a sanity count of RankDeficient rows (seeded data has none).
    n_bad = int(st.sum().item())

    # ---- roofline of the dominant kernel, timed per launch with CUDA events on its own stream
    int8_ms = statistics.mean(t["int8_ms"] for t in timing)
    fp64_ms = statistics.mean(t["fp64_ms"] for t in timing)
    conv_ms = statistics.mean(t["conv_ms"] for t in timing)
    int8_ms, fp64_ms, conv_ms, kern_avg_ms = multi.max_over_ranks([int8_ms, fp64_ms, conv_ms, kern_avg_ms],
                                                                  dist, device="cuda")
    flops_per_launch = float(n) * n * m * pR          # FP64 trsm flops, n^2 per X_R column (north star)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("config%d" % args.config)
        except Exception:
            traffic = None
    paths = timing[-1]["paths"]
    if paths[0] > 0:   # int8 digit-split path (integer genotypes)
        ops = OZ_SLICES * flops_per_launch           # int8 ops: 7 digit products per FP64 MAC
        peak, peak_sus, psrc = int8_peak()
        achieved = ops / (int8_ms / 1e3) / 1e12
        fp64eq = flops_per_launch / (int8_ms / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
                    "frac": achieved / peak, "traffic": traffic, "kernel": "ozaki_trsm_gls_kernel",
                    "kernel_ms": int8_ms,
                    "kernel_includes": "the FP64 -> int8 conversion of the next chunk's X_R (two convert-ahead "
                                       "warps, concurrent with the MMAs; only the first chunk's pass is separate)",
                    "fp64_fallback_ms": fp64_ms if paths[1] > 0 else 0.0,
                    "solve_block_ms": kern_avg_ms, "exposed_overhead_ms": kern_avg_ms - int8_ms,
                    "create_ms": statistics.mean(create_ms),
                    "int8_ops_per_launch": ops, "peak_source": psrc,
                    "frac_of_sustained_peak": achieved / peak_sus,
                    "fp64_equivalent": {"achieved_tflops": fp64eq, "dmma_peak_tflops": FP64_DMMA_PEAK_SUSTAINED,
                                        "ratio_to_dmma_peak": fp64eq / FP64_DMMA_PEAK_SUSTAINED,
                                        "note": "n^2 FP64 trsm flops per column / kernel time; the FP64 "
                                                "DMMA pipe peak is measured in profiles/r01_probe.txt"}}
    else:              # FP64 DMMA path
        achieved_tf = flops_per_launch / (fp64_ms / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": FP64_DMMA_PEAK_SUSTAINED,
                    "unit": "TFLOP/s", "frac": achieved_tf / FP64_DMMA_PEAK_SUSTAINED, "traffic": traffic,
                    "kernel": "fused_trsm_gls_kernel", "kernel_ms": fp64_ms, "solve_block_ms": kern_avg_ms,
                    "create_ms": statistics.mean(create_ms), "flops_per_launch": flops_per_launch,
                    "peak_source": "FP64 DMMA.8x8x4 microbenchmark on this pool's B200, 4 s sustained "
                                   "(profiles/r01_probe.txt); MEASURED_PEAKS.json has no FP64 entry"}

    # ---- e2e: the same job through the C ABI with HOST buffers, host<->device copies inside the
    # timed region (Alg. 8 double-buffered stream).  Primary: X_R as genotype codes (int8, one byte
    # per genotype -- gls_solve_block_i8); secondary: X_R as FP64 (gls_solve_block, 8 bytes).
    e2e = None
    if not args.no_e2e:
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except (ValueError, OSError):
            avail = 1 << 40
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        Mh = torch.from_numpy(P.M).pin_memory()
        XLh = torch.from_numpy(np.ascontiguousarray(P.XL)).pin_memory()
        yh = torch.from_numpy(P.y).pin_memory()

        def timed_e2e(solve, m_e):
            bh = torch.empty((m_e, p), dtype=torch.float64, pin_memory=True)
            sh = torch.empty(m_e, dtype=torch.int32, pin_memory=True)

            def one():
                ctx = make_ctx(Mh, XLh, yh)
                solve(ctx, m_e, bh, sh)
                ctx.close()

            one()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                one()
            torch.cuda.synchronize()
            dt = multi.max_over_ranks([(time.perf_counter() - t0) / args.steps], dist, device="cuda")[0]
            return dt, bool(torch.equal(bh, b[:m_e].cpu()))

        # int8 genotype codes: m x n bytes per rank
        m_i8 = int(min(m, 0.6 * avail / local_world / (n * pR)))
        m_i8 = max(m_i8 - m_i8 % 64, 64)
        Gh = torch.empty((m_i8 * pR, n), dtype=torch.int8, pin_memory=True)
        for c in range(0, m_i8 * pR, chunk):
            k = min(chunk, m_i8 * pR - c)
            Gh[c:c + k].copy_(Xd[c:c + k].to(torch.int8))
        dt8, same8 = timed_e2e(lambda ctx, me, bh, sh: ctx.solve_block_i8(Gh, me, bh, sh), m_i8)
        del Gh
        e2e = {"value": world * m_i8 / dt8, "unit": UNIT,
               "h2d_bytes_per_step": int((n * n + n * (pL + 1)) * 8 + m_i8 * pR * n),
               "d2h_bytes_per_step": int(m_i8 * p * 8 + m_i8 * 4),
               "m_per_rank": m_i8,
               "path": "C ABI gls_solve_block_i8: M, X_L, y (FP64) and X_R as int8 genotype codes in pinned "
                       "host memory -> double-buffered H2D stream; b and status back to pinned host memory",
               "bitwise_equal_to_device_run": same8}
        # FP64 X_R from host (8 bytes per genotype over PCIe), on at most 250k SNPs per rank (20 GB
        # pinned per rank at n = 1e4: a secondary number, kept cheap for the multi-GPU runs)
        m_f = int(min(m, 250_000, 0.6 * avail / local_world / (n * pR * 8)))
        m_f = max(m_f - m_f % 64, 64)
        Xh = torch.empty((m_f * pR, n), dtype=torch.float64, pin_memory=True)
        for c in range(0, m_f * pR, chunk):
            k = min(chunk, m_f * pR - c)
            Xh[c:c + k].copy_(Xd[c:c + k])
        dtf, samef = timed_e2e(lambda ctx, me, bh, sh: ctx.solve_block(Xh, me, bh, sh), m_f)
        del Xh
        e2e["fp64_host_input"] = {"value": world * m_f / dtf, "unit": UNIT, "m_per_rank": m_f,
                                  "h2d_bytes_per_step": int((n * n + n * (pL + 1) + m_f * pR * n) * 8),
                                  "d2h_bytes_per_step": int(m_f * p * 8 + m_f * 4),
                                  "path": "C ABI gls_solve_block, FP64 X_R in pinned host memory",
                                  "bitwise_equal_to_device_run": samef}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nsnp = 64 if n >= 5000 else 512
        L, t_chol, t_snp = oracle_sample(P, cfg, args.seed, nsnp)
        rate = nsnp / t_snp
        cpu = {"value": m / (t_chol + m / rate), "unit": UNIT, "cores": cpu_threads(), "kind": "oracle",
               "sample": "oracle Cholesky of the full n=%d M (%.2f s) + %d seeded SNPs of the workload "
                         "(%.2f s); value = m / (t_chol + m / rate)" % (n, t_chol, nsnp, t_snp)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "arithmetic": ("FP64 results; the trsm as exact int8 x int8 -> int32 digit products on tcgen05 "
                               "(T = L^-1 split into 7 base-256 digits, 55 bits per row; X_R integer) combined "
                               "and reduced in FP64 (DESIGN.md reading A15)") if roofline["kernel"].startswith("ozaki")
                              else "FP64 on the DMMA tensor pipe",
                "config": {"workload": "config%d: n=%d pL=%d pR=%d, %d SNPs per GPU in HBM (rank r owns "
                                       "SNPs [r*m, (r+1)*m))" % (args.config, n, pL, pR, m),
                           "n": n, "pL": pL, "pR": pR, "m_per_rank": m, "seed": args.seed,
                           "step": "gls_create (+NCCL broadcast) + gls_solve_block over all rank SNPs",
                           "l2": "inputs larger than L2 (X_R %.1f GB per rank)" % (m * pR * n * 8 / 1e9)},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches[0],
                "clocks": clk, "rank_deficient_rows": n_bad}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


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

    for _ in range(max(1, args.warmup)):
        step()
    clocks = ClockSampler(local)
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
