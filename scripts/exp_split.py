"""Time the ND coarse solve for several split levels (HH_ND_SPLIT) on a few grids."""
import os, subprocess, sys
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
import paper_2104_01439_b200.hh as hh
from workloads import config_spec
from workloads.configs import sweep_sample_spec
out = {}
for name, spec in [("cfg2", config_spec("cfg2")), ("n534", sweep_sample_spec({"id":0,"n":534,"k":160.0,"beta":0.5,"sigma":1.5})),
                   ("n268", sweep_sample_spec({"id":0,"n":268,"k":80.0,"beta":0.5,"sigma":1.5})),
                   ("n68", sweep_sample_spec({"id":0,"n":68,"k":20.0,"beta":0.5,"sigma":1.5}))]:
    gp = hh.Problem.from_spec(spec)
    r = torch.randn(gp.n_coarse, dtype=torch.complex128, device="cuda")
    e = gp.coarse_solve(r)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(50): gp.coarse_solve(r, e)
    t1.record(); torch.cuda.synchronize()
    out[name] = round(t0.elapsed_time(t1) / 50 * 1e3, 1)
    gp.close()
print(json.dumps(out))
'''
for cut in sys.argv[1:]:
    env = dict(os.environ)
    if cut != "auto":
        env["HH_ND_SPLIT"] = cut
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("split", cut, r.stdout.strip() or r.stderr[-800:])
