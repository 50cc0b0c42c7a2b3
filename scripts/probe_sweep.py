"""Sweep-share wall time (3 repeats) under the current env (HH_SWEEP_STREAMS ...)."""
import sys, time
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
for rep in range(3):
    t0 = time.perf_counter(); res = hh.sweep(s); t1 = time.perf_counter()
    dofs = sum(r["iterations"] * (x["n"] + 1) ** 2 for r, x in zip(res, s))
    print(f"rep {rep}: {t1 - t0:.3f} s  {dofs / (t1 - t0):.3e} it*DOF/s", flush=True)
