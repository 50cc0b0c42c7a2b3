"""ncu target for the roofline 'traffic' field (scripts/ncu_traffic.py).

  python scripts/traffic_target.py sweep|cfg2|cfg3 OUT.json

Runs the workload once unprofiled (plans, autotune, graphs, caches warm), then
once more inside cudaProfilerStart/Stop with the phase timers on, and writes the
timers (model / fused bytes and launches per phase) of that profiled pass to
OUT.json.  Run under
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      --clock-control none --csv --log-file L.csv python scripts/traffic_target.py ...
sweep = every 10th sample of the cfg1 sweep (352 samples: the same size and
shift mix as the full sweep), one engine stream so the kernels serialise."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01439_b200.hh as hh  # noqa: E402
import bench  # noqa: E402
from workloads import config_spec  # noqa: E402

what, out = sys.argv[1], sys.argv[2]
if what == "sweep":
    os.environ.setdefault("HH_SWEEP_STREAMS", "1")
    smp = bench.rank_samples(0, 1)[::10]
    o = hh.opts(restart=100, rtol=1e-6, max_iters=500)
    hh.sweep(smp, o=o)
    torch.cuda.synchronize()
    hh.sweep_timers(1)
    os.environ["HH_TIMING_EVERY"] = "1"
    torch.cuda.profiler.start()
    hh.sweep(smp, o=o)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    fl = hh.coarse_flops(None)[0]
    tm = hh.sweep_timers(0)
else:
    spec = config_spec(what)
    b = torch.from_numpy(spec.rhs()).cuda()
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    gp = hh.Problem.from_spec(spec)
    gp.fgmres_solve(b, o=o)
    torch.cuda.synchronize()
    gp.reset_timers(True)
    torch.cuda.profiler.start()
    gp.fgmres_solve(b, o=o)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    tm = gp.read_timers()
    fl = hh.coarse_flops(gp)[0]
    gp.close()
json.dump({"workload": what, "timers": tm, "coarse_flops": fl}, open(out, "w"))
print(json.dumps({k: tm[k] for k in hh.PHASES}))
