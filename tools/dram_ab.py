#!/usr/bin/env python
"""A/B: what the int8 kernel's DRAM traffic costs under the power cap.

Config-2 shape (n = 1e4, pL = 3, pR = 1, 1e6 SNPs in HBM).  The same solve two ways:
  fp64-in-HBM : gls_solve_block on FP64 X_R (the bench path): the kernel's convert-ahead warps read
                8 bytes per genotype of the next chunk and write 1 (plus the X8 panel re-reads)
  codes-in-HBM: gls_solve_block_i8 on int8 codes in HBM (ld % 16 == 0: read in place, no conversion)
and a third run with a short m (one wave of tiles, X8 panel = 190 MB) repeated, as a small-footprint
reference.  For each: CUDA-event time per solve, and nvidia-smi SM clock / power / throttle reasons
sampled every 50 ms during the timed loop.  Prints one JSON line.
"""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1210_7325_b200 as pkg  # noqa: E402


class Sampler:
    def __init__(self):
        self.rows, self.stop_ev = [], threading.Event()

    def run(self):
        p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
        while not self.stop_ev.is_set():
            line = p.stdout.readline()
            if not line:
                break
            self.rows.append([x.strip() for x in line.split(",")])
        p.terminate()

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join(timeout=2)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        pw = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        busy = [(s, w) for s, w in zip(sm, pw) if w > 500]
        return {"sm_mhz_median_under_load": statistics.median([s for s, _ in busy]) if busy else None,
                "power_w_median_under_load": statistics.median([w for _, w in busy]) if busy else None,
                "power_cap_samples": sum(1 for r in self.rows if len(r) > 2 and r[2].lower() == "active"),
                "samples": len(sm)}


def main():
    pkg.load()
    cfg = gen.CONFIGS[2]
    n, pL, pR = cfg.n, cfg.pL, cfg.pR
    m = 1_000_000
    P = gen.config_problem(cfg)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    X = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for c in range(0, m, 65536):
        k = min(65536, m - c)
        pkg.gen_xr_device(gen.DEFAULT_SEED, n, c, k, X[c:c + k])
    G = X.to(torch.int8)
    b = torch.empty((m, 4), dtype=torch.float64, device="cuda")
    out = {"workload": "config-2 shape, n=1e4, 1e6 SNPs in HBM"}
    with pkg.Context(n, pL, pR, d(P.M), d(P.XL), d(P.y)) as ctx:
        s = torch.cuda.Stream()
        ctx.set_stream(s.cuda_stream)
        wave = 148 * 128
        for name, fn, mm in (("fp64_in_hbm", lambda mm: ctx.solve_block(X, mm, b, None, async_=True), m),
                             ("codes_in_hbm", lambda mm: ctx.solve_block_i8(G, mm, b, None, async_=True), m),
                             ("codes_one_wave", lambda mm: ctx.solve_block_i8(G, mm, b, None, async_=True), wave)):
            reps = 5 if mm == m else 200
            fn(mm)
            ctx.sync()
            with Sampler() as smp:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(reps):
                    fn(mm)
                e1.record(s)
                ctx.sync()
                e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out[name] = {"m": mm, "ms_per_solve": ms, "snps_per_s": mm / ms * 1e3,
                         "int8_tops": 7.0 * n * n * mm / (ms * 1e-3) / 1e12, **smp.summary()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
