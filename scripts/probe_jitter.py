"""Host-side breakdown of repeated cfg2 steps (setup / solve / close) to find jitter."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
spec = config_spec("cfg2")
b = torch.from_numpy(spec.rhs()).cuda()
o = hh.opts(restart=spec.restart, rtol=spec.rtol)
for rep in range(20):
    t0 = time.perf_counter()
    gp = hh.Problem.from_spec(spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    x, r = gp.fgmres_solve(b, o=o)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    gp.close()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"rep {rep:2d} setup {1e3*(t1-t0):7.1f} solve {1e3*(t2-t1):7.1f} (dev {1e3*r['solve_s']:6.1f}) close {1e3*(t3-t2):6.1f} ms", flush=True)
