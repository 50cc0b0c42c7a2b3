"""Sweep-share wall time (6 repeats after warm-up) under the current env (HH_SWEEP_STREAMS ...)."""
import sys, time
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
hh.sweep(s)
ts = []
for rep in range(6):
    t0 = time.perf_counter(); res = hh.sweep(s); t1 = time.perf_counter()
    ts.append(t1 - t0)
dofs = sum(r["iterations"] * (x["n"] + 1) ** 2 for r, x in zip(res, s))
ts.sort()
print(f"sweep wall min {ts[0]:.3f} med {ts[3]:.3f} max {ts[-1]:.3f} s  -> {dofs / ts[3]:.3e} it*DOF/s (median)", flush=True)
