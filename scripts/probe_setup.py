"""Wall-time breakdown of repeated setup + solve (cfg2) and of a sweep group."""
import sys, time, json, os
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec, sweep_samples
spec = config_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
b = torch.from_numpy(spec.rhs()).cuda()
for rep in range(3):
    t0 = time.perf_counter()
    gp = hh.Problem.from_spec(spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    x, r = gp.fgmres_solve(b, o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    gp.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(json.dumps({"rep": rep, "setup": t1 - t0, "solve": t2 - t1, "close": t3 - t2, "its": r["iterations"]}))
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
for rep in range(2):
    t0 = time.perf_counter(); res = hh.sweep(s); t1 = time.perf_counter()
    print("sweep share", rep, t1 - t0, sum(r["iterations"] for r in res))
