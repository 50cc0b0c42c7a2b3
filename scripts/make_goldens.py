#!/usr/bin/env python
"""Write the oracle goldens for the full-size parity tests.  ORACLE-ONLY:
imports `oracle/` and `workloads/` and nothing from the CUDA path.

  python scripts/make_goldens.py cfg1 [--workers 6]      # all 3,520 sweep samples
  python scripts/make_goldens.py cfg2 | cfg3 | cfg4m      # full-size single solves

cfg1  -> tests/golden/cfg1_oracle.jsonl: one record per sample (id, n, k, sigma,
         beta, iterations, converged, rel_res_true, rho) of the oracle's
         FGMRES(100), rtol 1e-6, x0 = 0, point source at the centre
         (BASELINE configs[1]; Sec. 5 data generation),
         sample-parallel over host processes (one sample per process).
cfg2/cfg3/cfg4m -> tests/golden/<name>.json: for BASELINE configs[2] (1025^2),
         configs[3] (129^3) and the configs[4] medium at n = 128 (the "129^3
         analogue" of SURVEY.md 8(d)):
           coarse  e = A_eps^(1)^-1 r           (r = random_complex(Nc, 101))
           vcycle  z = V(f)                      (f = random_complex(N, 102))
           fgmres  iterations, converged, rel_res_true, rho and x
         each vector as its values at seeded sampled nodes plus four seeded
         projections w_k^H v (w_k = random_complex(len, 200 + k)), so a GPU
         error anywhere in the vector shows (Alg. 1).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.solve import OracleProblem  # noqa: E402
from workloads import config_spec, sweep_samples  # noqa: E402
from workloads.configs import sweep_sample_spec  # noqa: E402
from workloads.vectors import random_complex, sampled_nodes  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
N_SAMPLED = 2000
N_PROJ = 4


def _spec(name):
    if name == "cfg4m":
        return config_spec("cfg4", n=128)
    return config_spec(name)


def _cx(v):
    return [[float(a.real), float(a.imag)] for a in v]


def _vec_record(v, nodes, seed_base=200):
    proj = [complex(np.vdot(random_complex(v.size, seed_base + k), v)) for k in range(N_PROJ)]
    return {"nodes": [int(i) for i in nodes], "values": _cx(v[nodes]),
            "norm2": float(np.linalg.norm(v)), "proj": _cx(proj)}


def single(name):
    spec = _spec(name)
    t0 = time.perf_counter()
    op = OracleProblem(spec)
    t_setup = time.perf_counter() - t0
    print(f"{name}: setup {t_setup:.1f} s ({op.tg.coarse.kind})", flush=True)
    Nc = spec.n_coarse_nodes
    cnodes = sampled_nodes(spec.n // 2, spec.dim, N_SAMPLED, seed=301)
    fnodes = sampled_nodes(spec.n, spec.dim, N_SAMPLED, seed=302)
    b = spec.rhs()
    src = np.nonzero(b)[0]
    fnodes = np.unique(np.concatenate([fnodes, src]))
    r = random_complex(Nc, 101)
    e = op.tg.coarse.solve(r)
    f = random_complex(spec.n_nodes, 102)
    t1 = time.perf_counter()
    z = op.vcycle(f)
    t_vc = time.perf_counter() - t1
    t1 = time.perf_counter()
    x, rep = op.solve(b)
    t_solve = time.perf_counter() - t1
    print(f"{name}: vcycle {t_vc:.1f} s, solve {t_solve:.1f} s, {rep.iterations} its", flush=True)
    out = {
        "what": f"oracle goldens for {name} (scripts/make_goldens.py; oracle/ only)",
        "spec": {"name": spec.name, "dim": spec.dim, "n": spec.n, "k_const": spec.k_const,
                 "beta": spec.beta, "sigma": spec.sigma, "restart": spec.restart,
                 "rtol": spec.rtol, "max_iters": spec.max_iters, "source": list(spec.source)},
        "coarse_solver": op.tg.coarse.kind,
        "seeds": {"coarse_r": 101, "vcycle_f": 102, "proj_base": 200,
                  "coarse_nodes": 301, "fine_nodes": 302, "n_sampled": N_SAMPLED},
        "coarse": _vec_record(e, cnodes),
        "vcycle": _vec_record(z, fnodes),
        "fgmres": {"iterations": rep.iterations, "converged": bool(rep.converged),
                   "rel_res_true": rep.rel_res_true, "rho": rep.rho,
                   "restarts": rep.restarts, "x": _vec_record(x, fnodes)},
        "oracle_seconds": {"setup": t_setup, "vcycle": t_vc, "solve": t_solve},
    }
    path = os.path.join(GOLD, f"{name}_oracle.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path, flush=True)


def _one(s):
    t0 = time.perf_counter()
    _, rep = OracleProblem(sweep_sample_spec(s)).solve()
    return {"id": s["id"], "n": s["n"], "k": s["k"], "kh_target": s["kh_target"],
            "sigma": s["sigma"], "beta": s["beta"], "iterations": rep.iterations,
            "converged": bool(rep.converged), "rel_res_true": rep.rel_res_true, "rho": rep.rho,
            "seconds": time.perf_counter() - t0}


def cfg1(workers):
    from multiprocessing import Pool
    samples = sweep_samples()
    part = os.path.join(GOLD, "cfg1_oracle.partial.jsonl")
    done = {}
    if os.path.exists(part):
        for line in open(part):
            r = json.loads(line)
            done[r["id"]] = r
    todo = [s for s in samples if s["id"] not in done]
    # largest (n, shift strength) first so the pool drains evenly
    todo.sort(key=lambda s: -(s["n"] ** 2) * (1 + s["beta"] * s["k"] ** s["sigma"] / s["k"] ** 2))
    t0 = time.perf_counter()
    with open(part, "a") as fh, Pool(workers) as pool:
        for i, r in enumerate(pool.imap_unordered(_one, todo, chunksize=1)):
            done[r["id"]] = r
            fh.write(json.dumps(r) + "\n")
            fh.flush()
            if i % 50 == 0:
                print(f"{len(done)}/{len(samples)} after {time.perf_counter() - t0:.0f} s", flush=True)
    path = os.path.join(GOLD, "cfg1_oracle.jsonl")
    with open(path, "w") as fh:
        for s in samples:
            r = dict(done[s["id"]])
            r.pop("seconds", None)
            fh.write(json.dumps(r) + "\n")
    os.remove(part)
    print("wrote", path, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["cfg1", "cfg2", "cfg3", "cfg4m"])
    ap.add_argument("--workers", type=int, default=max(1, (os.cpu_count() or 2) - 2))
    a = ap.parse_args()
    if a.what == "cfg1":
        cfg1(a.workers)
    else:
        single(a.what)
