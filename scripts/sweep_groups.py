"""Per-group structure of a sweep share: B, iteration spread, batch solve time."""
import sys, collections
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
hh.sweep(s)
res = hh.sweep(s)
g = collections.defaultdict(list)
for r, x in zip(res, s):
    g[x["n"]].append((r["iterations"], r["solve_s"], r["setup_s"]))
tot = 0
for n in sorted(g):
    its = [a for a, _, _ in g[n]]
    t = max(b for _, b, _ in g[n]); su = max(c for _, _, c in g[n])
    tot += t
    print(f"n={n:4d} B={len(its):3d} its min {min(its):4d} max {max(its):4d} sum {sum(its):6d}  batch solve {t*1e3:8.2f} ms setup {su*1e3:7.2f} ms  ms/it {t*1e3/max(its):6.3f}")
print("sum of batch solve times", tot)
