"""cfg4 at full size (257^3 fine nodes, 129^3 coarse) on one GPU: setup, memory, one solve."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t0 = time.perf_counter()
spec = config_spec("cfg4", n=n)
t1 = time.perf_counter()
print("spec", n, spec.n_nodes, f"{t1 - t0:.1f} s", flush=True)
gp = hh.Problem.from_spec(spec)
torch.cuda.synchronize()
t2 = time.perf_counter()
free, tot = torch.cuda.mem_get_info()
print(f"setup {t2 - t1:.1f} s, device memory used {(tot - free) / 1e9:.1f} of {tot / 1e9:.1f} GB", flush=True)
b = torch.from_numpy(spec.rhs()).cuda()
for rep in range(2):
    t3 = time.perf_counter()
    x, r = gp.fgmres_solve(b, o=hh.opts(restart=spec.restart, rtol=spec.rtol))
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(json.dumps({"rep": rep, "solve_s": t4 - t3, **r, "itdof_per_s": r["iterations"] * spec.n_nodes / (t4 - t3)}), flush=True)
gp.close()
