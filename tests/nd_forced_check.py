"""Run by tests/test_gpu_nd_forced.py in a subprocess whose environment forces
the ND solve variants (the schedule switches are read once per process):
coarse solve, V-cycle and FGMRES parity against the oracle on small 3D grids.
Prints one JSON line of the worst errors."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])

import paper_2104_01439_b200.hh as hh  # noqa: E402
from oracle.solve import OracleProblem  # noqa: E402
from workloads import config_spec  # noqa: E402
from workloads.vectors import random_complex  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def specs():
    out = []
    for n in (8, 14, 18, 22):
        s = config_spec("cfg3", n=n)
        s.k_const = 40.0 * n / 128          # cfg3's k h
        out.append(s)
    out.append(config_spec("cfg4", n=12))
    out.append(config_spec("cfg4", n=20))
    return out


def main():
    worst = {"coarse": 0.0, "coarse_res": 0.0, "vcycle": 0.0, "x": 0.0, "dits": 0}
    for spec in specs():
        orc = OracleProblem(spec)
        gp = hh.Problem.from_spec(spec, coarse_solver=hh.HH_COARSE_ND)   # the ND kernels under test
        r = random_complex(spec.n_coarse_nodes, 3)
        e = gp.coarse_solve(torch.from_numpy(r).cuda())
        torch.cuda.synchronize()
        e = e.cpu().numpy()
        worst["coarse"] = max(worst["coarse"], rel(e, orc.tg.coarse.solve(r)))
        worst["coarse_res"] = max(worst["coarse_res"], rel(orc.tg.Ac @ e, r))
        f = random_complex(spec.n_nodes, 4)
        z = gp.vcycle(torch.from_numpy(f).cuda()).cpu().numpy()
        worst["vcycle"] = max(worst["vcycle"], rel(z, orc.vcycle(f)))
        b = spec.rhs()
        xo, ro = orc.solve(b)
        x, rg = gp.fgmres_solve(torch.from_numpy(b).cuda(),
                                o=hh.opts(restart=spec.restart, rtol=spec.rtol))
        worst["dits"] = max(worst["dits"], abs(rg["iterations"] - ro.iterations))
        x, rg = gp.fgmres_solve(torch.from_numpy(b).cuda(),
                                o=hh.opts(restart=spec.restart, rtol=spec.rtol, fixed_iters=ro.iterations))
        worst["x"] = max(worst["x"], rel(x.cpu().numpy(), xo))
        gp.close()
    print(json.dumps(worst))


if __name__ == "__main__":
    main()
