"""compute-sanitizer target for the dataflow ND solve kernels (k_nd_flow_fwd /
k_nd_flow_bwd): a small 2D problem with the flow schedule forced on every level
(HH_ND_FLOW=1 HH_ND_CUT=-1 HH_ND_SPLIT=99), two solves."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01439_b200.hh as hh  # noqa: E402
from workloads import config_spec  # noqa: E402
os.environ.update({"HH_ND_FLOW": "1", "HH_ND_CUT": "-1", "HH_ND_SPLIT": "99"})
spec = config_spec("cfg2", n=48)
gp = hh.Problem.from_spec(spec)
b = torch.from_numpy(spec.rhs()).cuda()
for _ in range(2):
    x, r = gp.fgmres_solve(b, o=hh.opts(restart=100, rtol=1e-6))
torch.cuda.synchronize()
print("its", r["iterations"], r["rel_res_true"])
gp.close()
