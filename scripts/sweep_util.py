"""Sweep-share wall vs summed phase time (HH_TIMING_EVERY=1) at 1 and 8 streams."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import sweep_samples
s = [x for x in sweep_samples() if x["id"] % 8 == 0]
hh.sweep(s)
hh.sweep_timers(1)
t0 = time.perf_counter(); res = hh.sweep(s); t1 = time.perf_counter()
tm = hh.sweep_timers(0)
tot = sum(tm[p]["ms"] for p in hh.PHASES)
print(f"streams={os.environ.get('HH_SWEEP_STREAMS')} wall {t1-t0:.3f} s  phase sum {tot/1e3:.3f} s  "
      + " ".join(f"{p}={tm[p]['ms']/1e3:.3f}" for p in hh.PHASES) + f" launches {tm['launches']}")
