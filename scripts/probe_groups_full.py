"""Per-n-group wall time of the full cfg1 sweep (each group swept alone, 2nd call
timed): it*DOF/s per group and its share of the summed group time."""
import sys, time, collections
sys.path.insert(0, ".")
import torch
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
allS = sweep_samples()
g = collections.defaultdict(list)
for x in allS:
    g[x["n"]].append(x)
rows, tot = [], 0.0
for n in sorted(g):
    s = g[n]
    hh.sweep(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); res = hh.sweep(s); torch.cuda.synchronize(); t = time.perf_counter() - t0
    its = sum(r["iterations"] for r in res)
    rows.append((n, len(s), its, t, its * (n + 1) ** 2 / t))
    tot += t
for n, B, its, t, r in rows:
    print(f"n={n:4d} B={B:3d} its={its:6d} wall {t*1e3:8.2f} ms share {t/tot:6.3f}  {r:.3e} it*DOF/s  us/it-batch {t*1e6/(its/B):8.1f}")
print(f"sum of group walls {tot:.3f} s")
t0 = time.perf_counter(); hh.sweep(allS); torch.cuda.synchronize(); print(f"full sweep wall {time.perf_counter()-t0:.3f} s")
