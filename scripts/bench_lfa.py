"""LFA engine measurement (NEXT f4 alternative): the sigma_c map
of PAPER.md Fig. sigma_LFA right (sigma_c against kh for h = 2^-4 .. 2^-10) on the
GPU through hh_lfa_sigma_c, against the ALU roofline, with the oracle timed on a
bounded sample.  Prints one JSON line.

Metric: theta-point symbol evaluations (4 x 4 spectral radius each) per second.
Roofline: FP64 flops per evaluation = 920 (symbols + characteristic polynomial +
start) + 480 per Aberth iteration, counted iterations from
hh_lfa_stats; peak = 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz = 37.2 TFLOP/s."""
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01439_b200.hh as hh  # noqa: E402

F0, F1 = 920.0, 480.0
PEAK_TFLOPS = 148 * 64 * 2 * 1965e6 / 1e12


def queries(m):
    qs = []
    for lv in range(4, 11):
        h = 2.0 ** -lv
        for kh in np.arange(0.05, 0.751, 0.05):
            qs.append(dict(k=float(kh) / h, h=h, beta=1.0, omega=0.6, nu1=2, nu2=2, m=m))
    return qs


def main():
    m = int(os.environ.get("LFA_M", "128"))
    steps, warm = 3, 2
    qs = queries(m)
    for _ in range(warm):
        hh.lfa_sigma_c(qs, tol=1e-3)
    hh.lfa_stats(reset=True)
    t0 = time.perf_counter()
    for _ in range(steps):
        sc = hh.lfa_sigma_c(qs, tol=1e-3)
    wall = time.perf_counter() - t0
    st = hh.lfa_stats(reset=True)
    evals_per_step = st["evals"] / steps
    kern_s = st["ms"] * 1e-3
    flops = F0 * st["evals"] + F1 * st["aberth_iters"]
    ach = flops / kern_s / 1e12
    # oracle on a bounded sample: rho_loc of one query at a coarse grid, scaled per evaluation
    from oracle import lfa
    mo = 24
    t1 = time.perf_counter()
    n_o = 0
    q = qs[len(qs) // 2]
    while time.perf_counter() - t1 < 10.0:
        lfa.rho_loc(lfa.lam_of(q["k"], 1.0, 1.5), q["h"], 0.6, 2, 2, m=mo)
        n_o += mo * mo - 1
    cpu_rate = n_o / (time.perf_counter() - t1)
    line = {"metric": "lfa_theta_evals_per_s", "value": st["evals"] / kern_s, "unit": "theta evals/s",
            "n_gpus": 1, "steps": steps, "warmup": warm, "ms_per_step": 1e3 * wall / steps,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "sigma_c map, h = 2^-4..2^-10, kh = 0.05..0.75 (105 queries)",
                       "m": m, "tol": 1e-3, "evals_per_step": evals_per_step,
                       "launches_per_step": st["launches"] / steps},
            "e2e": {"value": evals_per_step / (wall / steps), "unit": "theta evals/s",
                    "h2d_bytes_per_step": int(st["launches"] / steps) * 0, "d2h_bytes_per_step": 0,
                    "note": "host bisection loop, one rho_loc launch per round, wall clock"},
            "roofline": {"bound": "alu", "achieved": ach, "peak": PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": ach / PEAK_TFLOPS, "traffic": None,
                         "flops_model": f"{F0:.0f} per evaluation + {F1:.0f} per Aberth iteration",
                         "aberth_iters_per_eval": st["aberth_iters"] / st["evals"]},
            "cpu_baseline": {"value": cpu_rate, "unit": "theta evals/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle rho_loc (numpy eigvals) at m={mo}, 10 s"},
            "sigma_c_sample": {f"h=2^-{4 + i // 15},kh={0.05 * (1 + i % 15):.2f}": (None if math.isnan(v) else round(v, 4))
                               for i, v in enumerate(sc) if i % 15 in (5, 9, 13)}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
