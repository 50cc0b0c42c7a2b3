"""Repeated sweeps of rank 0's share (crash / race check)."""
import sys
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
ref = None
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    res = hh.sweep(s)
    its = [r["iterations"] for r in res]
    if ref is None:
        ref = its
    assert its == ref, "iteration counts changed between sweeps"
print("ok", sum(ref))
