"""ncu target: one sweep group (all samples of one grid size in this rank's share)."""
import sys
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
n = int(sys.argv[1]) if len(sys.argv) > 1 else 534
s = [x for x in sweep_samples() if x["n"] == n and x["id"] % 8 == 0]
res = hh.sweep(s)
print(n, len(s), sum(r["iterations"] for r in res))
