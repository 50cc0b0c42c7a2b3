"""Small end-to-end workload for compute-sanitizer (2D, 3D, het, sweep batch)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec, sweep_samples
for spec in [config_spec("cfg0", n=16), config_spec("cfg2", n=20), config_spec("cfg3", n=8), config_spec("cfg4", n=6)]:
    gp = hh.Problem.from_spec(spec)
    b = torch.from_numpy(spec.rhs()).cuda()
    x, r = gp.fgmres_solve(b, o=hh.opts(restart=spec.restart, rtol=spec.rtol, max_iters=40))
    gp.apply_op(0, b); gp.vcycle(b)
    torch.cuda.synchronize()
    print(spec.name, spec.n, r["iterations"], r["rel_res_true"])
    gp.close()
s = [x for x in sweep_samples() if x["n"] in (18, 34)][:12]
res = hh.sweep(s, o=hh.opts(max_iters=30))
print("sweep", [r["iterations"] for r in res])
