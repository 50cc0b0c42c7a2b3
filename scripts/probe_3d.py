"""3D fine-kernel microbenchmark: A_eps x / A_0 x applies (z-marching or naive
kernels, chosen by HH_3D_NAIVE / HH_3D_MINB) and the V-cycle on cfg3 / cfg4 at full
size; CUDA-event times, model bytes 32 + c B/node (c = 16 (A_eps) / 8 (A_0)
per element when heterogeneous)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01439_b200.hh as hh  # noqa: E402
from workloads import config_spec  # noqa: E402

out = {}
for name in sys.argv[1:] or ["cfg3", "cfg4"]:
    spec = config_spec(name)
    gp = hh.Problem.from_spec(spec)
    x = torch.randn(spec.n_nodes, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    het = spec.k_fine is not None
    res = {}
    for op, lab, c in ((hh.HH_OP_AEPS, "apply_eps", 16), (hh.HH_OP_A0, "apply_a0", 8)):
        for _ in range(3):
            gp.apply_op(op, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            gp.apply_op(op, x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        by = (32 + (c if het else 0)) * spec.n_nodes
        res[lab] = {"ms": ms, "model_gbs": by / ms / 1e6, "frac": by / ms / 1e6 / 6557.4}
    z = torch.empty_like(x)
    for _ in range(2):
        gp.vcycle(x, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gp.vcycle(x, z)
    e1.record()
    torch.cuda.synchronize()
    res["vcycle_ms"] = e0.elapsed_time(e1) / 5
    out[name] = res
    gp.close()
    torch.cuda.empty_cache()
print(json.dumps({"env": {k: os.environ.get(k) for k in ("HH_3D_NAIVE", "HH_3D_MINB")}, "res": out}))
