"""Small deterministic target for ncu: one cfg setup + two FGMRES solves."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = config_spec(name)
gp = hh.Problem.from_spec(spec)
b = torch.from_numpy(spec.rhs()).cuda()
o = hh.opts(restart=spec.restart, rtol=spec.rtol)
for _ in range(2):
    x, r = gp.fgmres_solve(b, o=o)
torch.cuda.synchronize()
print(name, r)
gp.close()
