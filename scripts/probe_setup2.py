"""Setup/solve breakdown (run with HH_PROFILE_SETUP=2 HH_DEBUG=1): cfg2, cfg3, a sweep share."""
import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec, sweep_samples
for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    if name == "sweep":
        s = [x for x in sweep_samples() if x["id"] % 8 == 0]
        for rep in range(2):
            t0 = time.perf_counter(); res = hh.sweep(s); t1 = time.perf_counter()
            print(f"sweep rep {rep}: wall {t1-t0:.3f} s setup_sum {sum(r['setup_s'] for r in res):.3f} "
                  f"solve_sum(per batch) {sum(r['solve_s'] for r in res):.3f}", flush=True)
        continue
    spec = config_spec(name)
    b = torch.from_numpy(spec.rhs()).cuda()
    for rep in range(2):
        t0 = time.perf_counter()
        gp = hh.Problem.from_spec(spec)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        x, r = gp.fgmres_solve(b, o=hh.opts(restart=spec.restart, rtol=spec.rtol))
        torch.cuda.synchronize(); t2 = time.perf_counter()
        gp.close(); torch.cuda.synchronize(); t3 = time.perf_counter()
        print(json.dumps({"cfg": name, "rep": rep, "setup": t1 - t0, "solve": t2 - t1, "close": t3 - t2,
                          "its": r["iterations"], "dev_solve": r["solve_s"]}), flush=True)
