"""Per-level ND solve timing (HH_ND_LEVEL_TIMING=1) of one coarse solve."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
spec = config_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
gp = hh.Problem.from_spec(spec)
r = torch.randn(gp.n_coarse, dtype=torch.complex128, device="cuda")
gp.coarse_solve(r)
torch.cuda.synchronize()
print("----", flush=True)
import os
os.environ["X"] = "1"
gp.coarse_solve(r)
torch.cuda.synchronize()
gp.close()
