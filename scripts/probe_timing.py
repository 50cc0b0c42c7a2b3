"""Quick timing probe (not the bench): cfg2 solve phases + a sweep subset."""
import time, json, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2104_01439_b200.hh as hh
from workloads import config_spec, sweep_samples

def run_cfg(name, n=None):
    spec = config_spec(name, n)
    t0 = time.perf_counter()
    gp = hh.Problem.from_spec(spec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    b = torch.from_numpy(spec.rhs()).cuda()
    o = hh.opts(restart=spec.restart, rtol=spec.rtol)
    x, r = gp.fgmres_solve(b, o=o)   # warm
    gp.reset_timers(True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    x, r = gp.fgmres_solve(b, o=o)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    tm = gp.read_timers()
    gp.reset_timers(False)
    x, r2 = gp.fgmres_solve(b, o=o)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    N = spec.n_nodes
    print(json.dumps({"cfg": name, "n": spec.n, "setup_s": t1 - t0, "iters": r["iterations"],
                      "solve_timed_s": t3 - t2, "solve_s": t4 - t3, "dev_solve_s": r2["solve_s"],
                      "itdof_per_s_solve": r2["iterations"] * N / (t4 - t3), "timers": tm,
                      "rel_res_true": r["rel_res_true"]}))
    gp.close()

run_cfg("cfg0")
run_cfg("cfg2", 256)
run_cfg("cfg2", 512)
run_cfg("cfg2")
s = sweep_samples()[::8]
t0 = time.perf_counter(); res = hh.sweep(s[:110]); t1 = time.perf_counter()
its = sum(r["iterations"] for r in res); dof = sum(r["iterations"] * (x["n"] + 1) ** 2 for r, x in zip(res, s))
print(json.dumps({"sweep_samples": len(res), "wall_s": t1 - t0, "iters": its, "itdof_per_s": dof / (t1 - t0),
                  "setup_s_sum": sum(r["setup_s"] for r in res), "solve_s_sum": sum(r["solve_s"] for r in res)}))
