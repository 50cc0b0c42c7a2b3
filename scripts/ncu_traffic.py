"""Per-phase DRAM traffic from an ncu launch list with dram metrics (the
roofline 'traffic' field of bench.py).

  python scripts/ncu_traffic.py LAUNCHES.csv TIMERS.json WORKLOAD [profiles/r02/traffic.json]

Classifies every profiled kernel into the FGMRES-iteration phases by name
(pre: k_pre*, k_jacobi3d/k_resid3d/k_restrict3d; coarse: the ND solve kernels;
post: k_post*, k_prolong3d, k_apply*; krylov: k_mdot*, k_update*, k_norm*,
k_trisolve, k_xupdate, k_advance, k_clear_jend; setup: factorisation and
coefficient kernels), sums dram__bytes_read.sum + dram__bytes_write.sum per
phase and divides by the phase's launch count from the timers of the same
profiled pass (one per batch iteration), next to the model bytes per launch."""
import collections
import csv
import json
import re
import sys

PHASE = [("coarse", r"^k_nd_(fwd|bwd|gather|rows_wide|fwdT|bwdK|bwd_stage|cluster|flow|fwd_sub|bwd_sub)"
                    r"|^k_fd_(fold|unfold|gemm)"),
         ("fine3d", r"^k_march3d|^k_bnd3d|^k_pw3d|^k_prolong3d"),   # 3D: shared by pre / post / A_0
         ("setup", r"^k_nd_|^k_fd_|^k_coef|^k_stencil|^k_dinv|^k_cstencil"),
         ("pre", r"^k_pre|^k_jacobi|^k_resid|^k_restrict"),
         ("post", r"^k_post|^k_prolong|^k_apply"),
         ("krylov", r"^k_mdot|^k_update|^k_norm|^k_trisolve|^k_xupdate|^k_advance|^k_clear_jend")]


def classify(name):
    for ph, rx in PHASE:
        if re.search(rx, name):
            return ph
    return "other"


def load(path):
    import gzip
    fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = [r for r in csv.reader(fh) if len(r) > 10]
    hdr = rows[0]
    ki, ii, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        name = re.sub(r"^void ", "", r[ki])
        name = re.sub(r"\(.*", "", name).replace("<unnamed>::", "")
        name = re.sub(r"<.*", "", name)
        names[r[ii]] = name
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}[unit]
        per[r[ii]][r[mi]] = v * scale
    return names, per


def main():
    path, tpath, wl = sys.argv[1], sys.argv[2], sys.argv[3]
    outp = sys.argv[4] if len(sys.argv) > 4 else None
    names, per = load(path)
    tm = json.load(open(tpath))["timers"]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        ph = classify(names[i])
        a = agg[ph]
        a[0] += 1
        a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a[2] += m.get("gpu__time_duration.sum", 0)
    res = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     f"--clock-control none (serialised, cold cache), {path.split('/')[-1]}"}
    for ph in ("pre", "coarse", "post", "krylov"):
        n = tm[ph]["launches"]
        if n <= 0 or ph not in agg:
            continue
        k, by, t = agg[ph]
        res[ph] = {"dram_bytes_per_launch": by / n, "model_bytes_per_launch": tm[ph]["model"] / n,
                   "fused_bytes_per_launch": tm[ph]["bytes"] / n, "kernels": k, "phase_launches": int(n),
                   "ncu_us_per_launch": 1e6 * t / n, "ncu_dram_gbs": by / t / 1e9 if t > 0 else None}
    fdk = [i for i in per if re.match(r"^k_fd_(fold|unfold|gemm)", names[i])]
    if fdk and "coarse" in res:   # fast-diagonalisation coarse solve: tensor-bound GEMMs
        n = tm["coarse"]["launches"]
        t = sum(per[i].get("gpu__time_duration.sum", 0) for i in fdk)
        g = [i for i in fdk if names[i].startswith("k_fd_gemm")]
        tg = sum(per[i].get("gpu__time_duration.sum", 0) for i in g)
        fl = json.load(open(tpath)).get("coarse_flops", 0.0)
        res["coarse_fd"] = {"dram_bytes_per_launch": res["coarse"]["dram_bytes_per_launch"],
                            "flops_per_launch": fl / n if n else None,
                            "ncu_us_per_launch": 1e6 * t / n, "gemm_share": tg / t if t else None,
                            "ncu_tflops": fl / t / 1e12 if t else None,
                            "ncu_gemm_tflops": fl / tg / 1e12 if tg else None}
    if "fine3d" in agg:   # 3D: the marching kernels serve pre, post and the A_0 apply
        k, by, t = agg["fine3d"]
        n = tm["pre"]["launches"]
        pre, post = res.get("pre", {}), res.get("post", {})
        by += pre.get("dram_bytes_per_launch", 0) * n + post.get("dram_bytes_per_launch", 0) * n
        t += 1e-6 * n * (pre.get("ncu_us_per_launch", 0) + post.get("ncu_us_per_launch", 0))
        res["fine3d_pre_post"] = {"dram_bytes_per_iteration": by / n,
                                  "model_bytes_per_iteration": (tm["pre"]["model"] + tm["post"]["model"]) / n,
                                  "ncu_us_per_iteration": 1e6 * t / n, "ncu_dram_gbs": by / t / 1e9}
        res.pop("pre", None)
        res.pop("post", None)
    res["setup"] = {"kernels": agg["setup"][0], "dram_bytes": agg["setup"][1], "ncu_ms": 1e3 * agg["setup"][2]}
    tot_t = sum(a[2] for a in agg.values())
    res["time_share"] = {ph: round(a[2] / tot_t, 4) for ph, a in agg.items()} if tot_t else {}
    print(json.dumps(res, indent=1))
    if outp:
        try:
            allr = json.load(open(outp))
        except Exception:
            allr = {}
        allr[wl] = res
        json.dump(allr, open(outp, "w"), indent=1)


if __name__ == "__main__":
    main()
