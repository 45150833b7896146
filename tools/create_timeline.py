"""Diagnostics: kernel timeline of one gls_create (all streams) through the CUPTI activity records
torch.profiler collects.  Writes gpurun_out/create_timeline_n<N>.json: [name, stream, start_us,
dur_us, grid] per kernel.  usage: python tools/create_timeline.py [n]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import gen
import paper_1210_7325_b200 as pkg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
P = gen.make_problem(n, 3, 1)
Md, XLd, yd = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (P.M, P.XL, P.y))
for _ in range(3):
    pkg.Context(n, 3, 1, Md, XLd, yd).close()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    c = pkg.Context(n, 3, 1, Md, XLd, yd)
    torch.cuda.synchronize()
c.close()
os.makedirs("gpurun_out", exist_ok=True)
path = "gpurun_out/create_trace_n%d.json" % n
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") == "kernel"]
out = [[e["name"], e["args"].get("stream"), e["ts"], e["dur"], e["args"].get("grid")] for e in ks]
out.sort(key=lambda r: r[2])
json.dump(out, open("gpurun_out/create_timeline_n%d.json" % n, "w"))
t0 = out[0][2]
t1 = max(r[2] + r[3] for r in out)
print("n=%d: %d kernels, span %.3f ms" % (n, len(out), (t1 - t0) / 1e3))
