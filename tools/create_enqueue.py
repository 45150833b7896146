"""Diagnostics: host-side enqueue time of gls_create (gls_create_async returns after enqueueing every
step) vs the create's total time, with and without an nvidia-smi -lms 200 sampler running (bench.py's
clock sampler).  usage: python tools/create_enqueue.py [n]"""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
import paper_1210_7325_b200 as pkg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
P = gen.make_problem(n, 3, 1)
Md, XLd, yd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P.M, P.XL, P.y))
for smi in (False, True, False):
    p = (subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader",
                           "-lms", "200"], stdout=subprocess.DEVNULL) if smi else None)
    time.sleep(0.5)
    enq, tot, syn = [], [], []
    for r in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = pkg.Context(n, 3, 1, Md, XLd, yd, async_create=True)
        t1 = time.perf_counter()
        c.sync()
        t2 = time.perf_counter()
        c.close()
        t0b = time.perf_counter()
        c = pkg.Context(n, 3, 1, Md, XLd, yd)
        t3 = time.perf_counter()
        c.close()
        enq.append(1e3 * (t1 - t0)); tot.append(1e3 * (t2 - t0)); syn.append(1e3 * (t3 - t0b))
    if p:
        p.terminate()
    print("smi=%d  async enqueue %s ms | async total %s | sync create %s" % (
        smi, " ".join("%.1f" % v for v in enq[1:]), " ".join("%.1f" % v for v in tot[1:]),
        " ".join("%.1f" % v for v in syn[1:])), flush=True)
