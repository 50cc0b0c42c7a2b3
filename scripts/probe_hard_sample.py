"""The sweep's critical path: the hardest n = 534 sample of rank 0's share, solved alone."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
from workloads.configs import sweep_sample_spec
s = [x for x in sweep_samples() if x["id"] % 8 == 0 and x["n"] == 534]
hard = max(s, key=lambda x: x["beta"] * x["k"] ** x["sigma"])
spec = sweep_sample_spec(hard)
gp = hh.Problem.from_spec(spec)
b = torch.from_numpy(spec.rhs()).cuda()
o = hh.opts(restart=100, rtol=1e-6)
x, r = gp.fgmres_solve(b, o=o)
gp.reset_timers(True)
t0 = time.perf_counter(); x, r = gp.fgmres_solve(b, o=o); torch.cuda.synchronize(); t1 = time.perf_counter()
tm = gp.read_timers()
gp.reset_timers(False)
t2 = time.perf_counter(); x, r = gp.fgmres_solve(b, o=o); torch.cuda.synchronize(); t3 = time.perf_counter()
print(json.dumps({"sample": hard, "its": r["iterations"], "solve_timed_s": t1 - t0, "solve_s": t3 - t2,
                  "ms_per_it": 1e3 * (t3 - t2) / r["iterations"],
                  "phase_us_per_it": {p: 1e3 * tm[p]["ms"] / max(tm[p]["launches"], 1) for p in hh.PHASES}}))
