"""Sweep share: wall time of setup + 1 iteration (max_iters=1) vs the full solve,
at the current HH_SWEEP_STREAMS -- the setup share of a sweep step."""
import sys, time
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
for name, o in (("max_iters=1", hh.opts(max_iters=1)), ("full", None)):
    hh.sweep(s, o=o)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); hh.sweep(s, o=o); ts.append(time.perf_counter() - t0)
    print(f"{name}: median {sorted(ts)[2]:.3f} s", flush=True)
