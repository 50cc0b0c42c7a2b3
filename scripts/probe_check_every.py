"""Sweep share wall time at several host polling intervals (check_every)."""
import sys, time
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
for ce in (1, 4, 16):
    o = hh.opts(restart=100, rtol=1e-6, max_iters=500, check_every=ce)
    hh.sweep(s, o=o)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); res = hh.sweep(s, o=o); ts.append(time.perf_counter() - t0)
    its = sum(r["iterations"] for r in res)
    print(f"check_every={ce}: median {sorted(ts)[2]:.4f} s, iterations {its}", flush=True)
