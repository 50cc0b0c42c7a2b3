"""FD coarse-solve throughput per grid size at the sweep's real batch sizes.

  python scripts/probe_fd.py [n ...]

For every n: all cfg1 samples with that n (110, or 220 when two (k, kh) classes
share it) through hh_sweep on ONE engine stream with every iteration timed,
then the coarse phase's average per-launch time and TFLOP/s (hh_coarse_flops),
next to the other phases.  Diagnostics only."""
import json
import os
import sys

os.environ["HH_SWEEP_STREAMS"] = "1"
os.environ["HH_TIMING_EVERY"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2104_01439_b200.hh as hh  # noqa: E402
from workloads import sweep_samples  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [34, 68, 134, 200, 268, 400, 534]
allsmp = sweep_samples()
o = hh.opts(restart=100, rtol=1e-6, max_iters=500)
for n in ns:
    smp = [s for s in allsmp if s["n"] == n]
    if not smp:
        continue
    hh.sweep(smp, o=o)                      # warm (engines, graphs)
    torch.cuda.synchronize()
    hh.sweep_timers(1)
    hh.sweep(smp, o=o)
    torch.cuda.synchronize()
    fl = hh.coarse_flops(None)
    tm = hh.sweep_timers(0)
    row = {"n": n, "samples": len(smp), "P": n // 4 + 1}
    for ph in hh.PHASES:
        d = tm[ph]
        if d["launches"]:
            row[ph + "_us"] = round(1e3 * d["ms"] / d["launches"], 1)
    c = tm["coarse"]
    row["coarse_tflops"] = round(fl[0] / (c["ms"] * 1e-3) / 1e12, 2) if c["ms"] > 0 else None
    row["coarse_share"] = round(c["ms"] / sum(tm[p]["ms"] for p in hh.PHASES), 3)
    print(json.dumps(row), flush=True)
