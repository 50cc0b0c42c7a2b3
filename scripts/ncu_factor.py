"""ncu target: the coarse factorisation of one problem (setup only)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
spec = config_spec(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
gp = hh.Problem.from_spec(spec)
torch.cuda.synchronize()
gp.close()
