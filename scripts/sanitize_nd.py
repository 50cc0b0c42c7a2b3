"""compute-sanitizer target: a small 3D solve whose top fronts take the
global-memory (f > vmax) and wide ND paths (run with HH_ND_VMAX=200)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
spec = config_spec("cfg3", n=32)
spec.k_const = 10.0
gp = hh.Problem.from_spec(spec)
x, r = gp.fgmres_solve(torch.from_numpy(spec.rhs()).cuda(), o=hh.opts(restart=50, rtol=1e-6))
torch.cuda.synchronize()
print("its", r["iterations"], r["rel_res_true"])
gp.close()
