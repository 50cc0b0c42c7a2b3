"""Per-rank sweep time of every shard, measured one shard at a time on ONE GPU
(the ranks of a multi-GPU sweep are independent: no collective on the data
path, one record gather at the end), for round-robin and group-aware sharding.

  python scripts/probe_shards.py [world ...]

Prints, per (world, sharding), every shard's device time (CUDA events around
hh_sweep, warm engines, L2 flushed), max / mean, and the implied step time and
scaling efficiency T(1) / (world * max shard time).  An estimate of the N-GPU
step from N single-GPU measurements -- not a multi-GPU run."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2104_01439_b200.hh as hh  # noqa: E402
import bench  # noqa: E402

worlds = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
o = hh.opts(restart=100, rtol=1e-6, max_iters=500)
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")


def timed(samples, reps=2):
    hh.sweep(samples, o=o)
    best = None
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hh.sweep(samples, o=o)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


t1 = timed(bench.rank_samples(0, 1))
print(json.dumps({"world": 1, "ms": round(t1, 1)}), flush=True)
for w in worlds:
    for sh in ("roundrobin", "groups"):
        ms = [timed(bench.rank_samples(r, w, sh)) for r in range(w)]
        mx = max(ms)
        print(json.dumps({"world": w, "sharding": sh, "shard_ms": [round(x, 1) for x in ms],
                          "max_ms": round(mx, 1), "mean_ms": round(sum(ms) / w, 1),
                          "efficiency": round(t1 / (w * mx), 3)}), flush=True)
