"""Per-level factorisation timing (HH_PROFILE_SETUP=2) of the largest sweep grid."""
import sys
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
n = int(sys.argv[1]) if len(sys.argv) > 1 else 534
s = [x for x in sweep_samples() if x["id"] % 8 == 0 and x["n"] == n][:4]
hh.sweep(s)
print("---", flush=True)
hh.sweep(s)
