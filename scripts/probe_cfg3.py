import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
spec = config_spec(name, n)
t0 = time.perf_counter()
gp = hh.Problem.from_spec(spec)
torch.cuda.synchronize(); t1 = time.perf_counter()
print("setup_s", t1 - t0, "mem GB", torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, flush=True)
b = torch.from_numpy(spec.rhs()).cuda()
for rep in range(2):
    t1 = time.perf_counter()
    x, r = gp.fgmres_solve(b, o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(json.dumps({"name": name, "n": spec.n, "solve_s": t2 - t1, **r, "itdof": r["iterations"] * spec.n_nodes / (t2 - t1)}), flush=True)
