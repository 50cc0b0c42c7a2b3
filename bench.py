#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: preconditioned FGMRES
iterations x DOF / s, complex fp64, and HBM GB/s vs peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload sweep|search|cfg0|cfg2|cfg3|cfg4]

Workloads:
  sweep (default, BASELINE configs[1]): a step = the WHOLE 3,520-sample shift
        sweep.  At N ranks every rank takes a 1/N share: the samples sorted by
        (grid size, shift strength beta k^sigma) are dealt round-robin, so every
        rank gets the same mix of sizes and expected iteration counts (strong
        scaling: total work fixed).  Every sample is set up, its coarse operator
        factored, and solved (point source, FGMRES(100), rtol 1e-6) inside the
        step, as the paper's end-to-end times do; at N > 1 the
        per-sample records are gathered to rank 0 inside the step.
  cfg2 / cfg0 / cfg3 / cfg4: a step = setup + factorisation + one full solve of
        that config (slab-decomposed over the ranks at N > 1).
value = sum over ranks of iterations x fine DOFs / max-over-ranks device time.
No oracle code runs on the product arm except the bounded cpu_baseline leg
(rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import config_spec, sweep_samples  # noqa: E402
from workloads.configs import sweep_sample_spec  # noqa: E402

METRIC = "preconditioned FGMRES iterations*DOF/s (complex fp64)"
SEARCH_COUNT, SEARCH_LEVELS = 48, (4, 5, 6, 7, 8, 9)
UNIT = "it*DOF/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """SM clock and throttle-reason sampler (NVML, every 100 ms, in a thread of
    this process: only the SM clock and the clocks-event-reason bits are read,
    which do not stall concurrent CUDA calls the way an nvidia-smi process polling
    the full query set did).  Started before the warm-up; only the samples inside
    the timed region [mark(), stop()] are reported.  Falls back to nvidia-smi if
    NVML cannot be loaded."""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4))

    def __init__(self, dev):
        import threading
        self.t0 = None
        self.rows = []
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = dev
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[dev])
                except ValueError:
                    idx = dev
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    def _run(self):
        nv = self.nv
        while not self.stop_ev.wait(0.1):
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((time.time(), float(sm), rs))
            except Exception:
                pass

    def mark(self):
        """Start of the timed region."""
        self.t0 = time.time()

    def stop(self):
        if not self.ok:
            return None
        t1 = time.time()
        self.stop_ev.set()
        self.th.join(timeout=2)
        rows = [r for r in self.rows if self.t0 is None or self.t0 - 0.05 <= r[0] <= t1 + 0.05]
        if not rows:
            return None
        sm = sorted(r[1] for r in rows)
        reasons = sorted({n for r in rows for n, bit in self.NAMES if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.max), "samples": len(rows),
                "reasons": reasons, "source": "nvml"}


def rank_samples(rank, world, sharding="groups"):
    """This rank's 1/world share of the whole sweep; world = 1 is the full
    3,520-sample sweep.
      roundrobin: samples sorted by (grid size n, shift strength beta k^sigma, id)
        are dealt round-robin, so every rank gets the same mix of grid sizes and
        (expected) iteration counts;
      groups: grids with (n+1)^2 >= 2.4e6 / 110 (the node budget already cuts
        their 110-sample groups into several batches on one GPU) are dealt
        round-robin as above; every smaller grid's group stays WHOLE on one rank
        (its lockstep batch keeps all 110 / 220 samples, as on one GPU), the
        groups placed largest-first on the least-loaded rank (fine nodes)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    order = sorted(sweep_samples(), key=lambda s: (s["n"], s["beta"] * s["k"] ** s["sigma"], s["id"]))
    if sharding == "roundrobin" or world == 1:
        return [s for p, s in enumerate(order) if p % world == rank]
    if sharding != "groups":
        raise ValueError(f"unknown sharding {sharding!r}")
    split = 2.4e6 / 110
    big = [s for s in order if (s["n"] + 1) ** 2 >= split]
    mine = [s for p, s in enumerate(big) if p % world == rank]
    load = [0.0] * world
    for p, s in enumerate(big):
        load[p % world] += (s["n"] + 1) ** 2
    groups = {}
    for s in order:
        if (s["n"] + 1) ** 2 < split:
            groups.setdefault(s["n"], []).append(s)
    for n, g in sorted(groups.items(), key=lambda kv: (-len(kv[1]) * (kv[0] + 1) ** 2, kv[0])):
        r = min(range(world), key=lambda q: (load[q], q))
        load[r] += len(g) * (n + 1) ** 2
        if r == rank:
            mine.extend(g)
    return mine


def gather_records(res, world):
    """Per-sample records of every rank, gathered to all ranks (one
    all_gather_object; the only data exchange of the sweep), sorted by id."""
    recs = [(r["id"], r["status"], r["iterations"], r["converged"], r["rel_res_true"], r["rho"])
            for r in res]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, recs)
        recs = [x for part in allr for x in part]
    return sorted(recs)


def combine_ranks(dev_ms, dofs, its, world, device):
    """Max over ranks of the device time, sum over ranks of the work (the
    only collective of the bench; none on the data path)."""
    t = torch.tensor([dev_ms, float(dofs), float(its)], dtype=torch.float64, device=device)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        return tmax[0].item(), tsum[1].item(), tsum[2].item()
    return dev_ms, float(dofs), float(its)


def share_nccl_id(make_id, rank, device):
    """Rank 0's 128-byte NCCL id, broadcast over the default process group."""
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.tensor(list(make_id()), dtype=torch.uint8))
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


def slab_part(vec, n, dim, z, rank):
    """This rank's owned planes [z[rank], z[rank+1]) of a global fine vector."""
    plane = (n + 1) ** (dim - 1)
    return vec[z[rank] * plane: z[rank + 1] * plane]


# ------------------------------------------------------------------ ours
def run_ours(args, rank, world, dev):
    import paper_2104_01439_b200.hh as hh
    stream = torch.cuda.current_stream()
    if args.workload == "sweep":
        samples = rank_samples(rank, world, args.sharding)
        o = hh.opts(restart=100, rtol=1e-6, max_iters=500, check_every=args.check_every)
        gathered = {"recs": None}

        def step():
            res = hh.sweep(samples, o=o, coarse_solver=COARSE[args.coarse_solver])
            its = sum(r["iterations"] for r in res)
            dofs = sum(r["iterations"] * (s["n"] + 1) ** 2 for r, s in zip(res, samples))
            bad = [r for r in res if r["status"] != 0]
            if bad:
                raise RuntimeError(f"sweep sample failed: {bad[0]}")
            gathered["recs"] = gather_records(res, world)   # inside the step
            return its, dofs, res

        wl = {"workload": "cfg1 shift sweep (BASELINE configs[1]), all 3,520 samples",
              "samples_per_rank": len(samples), "samples_total": len(sweep_samples()),
              "sharding": args.sharding,
              "restart": 100, "rtol": 1e-6,
              "l2": "per-sample working sets are L2-resident; L2 flushed (512 MB write) between steps"}
    elif args.workload == "search":
        from workloads.configs import search_rhs, search_samples
        samples = [x for x in search_samples(SEARCH_COUNT, seed=0, levels=SEARCH_LEVELS)
                   if x["id"] % world == rank]
        rhs = [search_rhs(x, seed=0) for x in samples]

        def step():
            res = hh.shift_search(samples, rhs)
            its = sum(r["iterations_total"] for r in res)
            dofs = sum(r["iterations_total"] * (x["n"] + 1) ** 2 for r, x in zip(res, samples))
            return its, dofs, res

        wl = {"workload": "shift search (PAPER.md Sec. 5 steps 1-6, SURVEY 8(f) 1)",
              "samples_per_rank": len(samples), "levels": list(SEARCH_LEVELS), "tol": 1e-2,
              "budget": "rtol 1e-8 / 50 iterations", "rhs": "U[-1,1] per sample, seeded",
              "l2": "L2 flushed (512 MB write) between steps"}
    else:
        spec = config_spec(args.workload)
        slabkw = {}
        rhs = spec.rhs()
        if world > 1:
            # one solve, slab-decomposed over the ranks (NCCL halos + allreduces); the
            # coarse factor replicated (SURVEY 8(e) first version) or distributed
            # over the slabs (--coarse dist: HH_COARSE_ND_DIST)
            nid = share_nccl_id(hh.nccl_unique_id, rank, dev)
            z = hh.slab_bounds(spec.n, world)
            rhs = slab_part(rhs, spec.n, spec.dim, z, rank)
            slabkw = {"nccl_id": nid, "rank": rank, "nranks": world}
            if args.coarse == "dist":
                slabkw["coarse_solver"] = hh.HH_COARSE_ND_DIST

        b_dev = torch.from_numpy(np.ascontiguousarray(rhs)).to(dev)
        timers = {"on": False, "acc": None, "flops": [0.0, 0.0], "kind": None}

        def step():
            kw = dict(slabkw)
            if args.coarse_solver != "auto" and "coarse_solver" not in kw:
                kw["coarse_solver"] = COARSE[args.coarse_solver]
            gp = hh.Problem.from_spec(spec, **kw)   # setup + coarse factorisation (inside the step)
            if timers["on"]:
                gp.reset_timers(True)
            x, r = gp.fgmres_solve(b_dev, o=hh.opts(restart=spec.restart, rtol=spec.rtol,
                                                     max_iters=spec.max_iters))
            if timers["on"]:
                t = gp.read_timers()
                if timers["acc"] is None:
                    timers["acc"] = t
                else:
                    for ph in hh.PHASES:
                        for key in ("ms", "bytes", "launches", "bytes_all", "model", "model_all"):
                            timers["acc"][ph][key] += t[ph][key]
                    timers["acc"]["launches"] += t["launches"]
                f = hh.coarse_flops(gp)
                timers["flops"][0] += f[0]
                timers["flops"][1] += f[1]
            timers["kind"] = gp.coarse_kind()
            gp.close()
            # one solve over all ranks: each rank counts its share of the work
            return r["iterations"] / world, r["iterations"] * spec.n_nodes / world, [r]

        wl = {"workload": f"{args.workload} (BASELINE configs[{args.workload[-1]}])",
              "n_cells": spec.n, "dim": spec.dim, "restart": spec.restart, "rtol": spec.rtol,
              "l2": "Krylov basis > L2 (126 MB); L2 flushed between steps",
              "parallelism": f"slab{world}" if world > 1 else "single",
              "coarse": None}
    flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device=dev)
    clk = Clocks(dev) if rank == 0 and not os.environ.get("HH_BENCH_NO_CLOCKS") else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if clk:
        clk.mark()
    if args.workload in ("sweep", "search"):
        hh.sweep_timers(1)
    else:
        timers["on"] = True
    ev = []
    tot_its = tot_dofs = 0
    results = []
    prof = bool(os.environ.get("HH_BENCH_PROFILE"))   # ncu --profile-from-start off: the timed steps only
    if prof:
        torch.cuda.profiler.start()
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        its, dofs, res = step()
        e1.record(stream)
        ev.append((e0, e1))
        tot_its += its
        tot_dofs += dofs
        results = res
    torch.cuda.synchronize()
    if prof:
        torch.cuda.profiler.stop()
    if world > 1:
        dist.barrier()
    clocks = clk.stop() if clk else None
    step_ms = [a.elapsed_time(b) for a, b in ev]
    print("step ms: " + " ".join(f"{x:.1f}" for x in step_ms), file=sys.stderr)
    dev_ms = sum(step_ms)
    rank_ms = [dev_ms]
    if world > 1:   # per-rank device time (load balance of the shards)
        rank_ms = [None] * world
        dist.all_gather_object(rank_ms, dev_ms)
    if args.workload in ("sweep", "search"):
        flops = hh.coarse_flops(None)        # before sweep_timers(0) resets them
        tm = hh.sweep_timers(0)
        wl["coarse"] = ("fast diagonalisation on every batch (HH_COARSE_AUTO: constant k, resolved "
                        "coarse grids; ND factor only on a validation failure)")
    else:
        timers["on"] = False
        tm = timers["acc"]
        flops = tuple(timers["flops"])
        kind = {hh.HH_COARSE_FD: "fast diagonalisation (FP64 tensor-core GEMMs)",
                hh.HH_COARSE_ND: "nested-dissection factor" + (" (replicated)" if world > 1 else ""),
                hh.HH_COARSE_ND_DIST: "distributed slab-aligned ND"}
        wl["coarse"] = kind.get(timers["kind"], str(timers["kind"]))
    if tm is not None:
        tm["coarse_flops"], tm["coarse_flops_all"] = flops[0], flops[1]
    dev_ms, tot_dofs, tot_its = combine_ranks(dev_ms, tot_dofs, tot_its, world, dev)
    value = tot_dofs / (dev_ms * 1e-3)
    out = {"value": value, "ms_per_step": dev_ms / args.steps, "wl": wl, "timers": tm,
           "clocks": clocks, "iterations_total": int(tot_its)}
    if world > 1:
        wl["rank_ms_per_step"] = [round(x / args.steps, 2) for x in rank_ms]
    if args.workload == "sweep":
        recs = gathered["recs"]
        wl["records_gathered"] = len(recs)
        wl["records_converged"] = sum(1 for r in recs if r[3])
        if rank == 0 and args.records:
            with open(args.records, "w") as fh:
                for r in recs:
                    fh.write(json.dumps({"id": r[0], "status": r[1], "iterations": r[2], "converged": r[3],
                                         "rel_res_true": r[4], "rho": r[5]}) + "\n")
    # e2e: same metric through the public API with host-side inputs/outputs each step
    if args.workload in ("sweep", "search"):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        its, dofs, _ = step()          # hh_sweep / hh_shift_search: host inputs in, host records out
        e2e_s = time.perf_counter() - t0
        e2e_s, dofs, _ = combine_ranks(e2e_s, dofs, its, world, dev)
        h2d = len(samples) * (40 + 16)
        if args.workload == "search":
            h2d = sum(16 * (x["n"] + 1) ** 2 for x in samples) * 12   # rhs per evaluation
        out["e2e"] = {"value": dofs / e2e_s, "unit": UNIT,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": len(samples) * 56}
    else:
        bh = torch.from_numpy(np.ascontiguousarray(rhs)).pin_memory().numpy()
        xh = torch.zeros(bh.size, dtype=torch.complex128).pin_memory().numpy()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        gp = hh.Problem.from_spec(spec, **slabkw)
        r = gp.fgmres_solve_host(bh, xh, hh.opts(restart=spec.restart, rtol=spec.rtol))
        gp.close()
        e2e_s = time.perf_counter() - t0
        if world > 1:
            e2e_s = combine_ranks(e2e_s, 0.0, 0.0, world, dev)[0]
        kb = 0 if spec.k_fine is None else 8 * (spec.k_fine.size + spec.k_coarse.size)
        out["e2e"] = {"value": r["iterations"] * spec.n_nodes / e2e_s, "unit": UNIT,
                      "h2d_bytes_per_step": 32 * bh.size + kb,     # b and x0, k_e arrays
                      "d2h_bytes_per_step": 16 * bh.size}
    if rank == 0 and world == 1 and not args.no_cold:
        out["e2e"]["cold"] = cold_probe(args)
    return out


def cold_probe(args):
    """One step of the same workload through the public API in a FRESH process
    (no ND plans, autotuned schedules, engines or device block caches yet):
    the first-call end-to-end time a new user sees (CUDA context creation
    excluded, timed from the first hh call)."""
    cmd = [sys.executable, os.path.abspath(__file__), "--cold-probe", "--workload", args.workload]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
        return json.loads(line)
    except Exception as e:   # reported, never fatal
        return {"error": f"{type(e).__name__}: {e}"[:200]}


def run_cold_probe(args):
    import paper_2104_01439_b200.hh as hh
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")                     # CUDA context outside the timed region
    torch.cuda.synchronize()
    if args.workload == "sweep":
        samples = rank_samples(0, 1)
        t0 = time.perf_counter()
        res = hh.sweep(samples, o=hh.opts(restart=100, rtol=1e-6, max_iters=500))
        dt = time.perf_counter() - t0
        dofs = sum(r["iterations"] * (s["n"] + 1) ** 2 for r, s in zip(res, samples))
        what = f"hh_sweep of all {len(samples)} samples, first call in a fresh process"
    else:
        spec = config_spec(args.workload)
        bh = np.ascontiguousarray(spec.rhs())
        xh = np.zeros_like(bh)
        t0 = time.perf_counter()
        gp = hh.Problem.from_spec(spec)
        r = gp.fgmres_solve_host(bh, xh, hh.opts(restart=spec.restart, rtol=spec.rtol))
        gp.close()
        dt = time.perf_counter() - t0
        dofs = r["iterations"] * spec.n_nodes
        what = "setup + factor + host-buffer solve, first call in a fresh process"
    print(json.dumps({"value": dofs / dt, "unit": UNIT, "seconds": dt, "what": what}))


# ------------------------------------------------------------------ oracle (CPU)
def _oracle_sweep_sample(s):
    """One cfg1 sample through the oracle (a pool worker): setup + LU + solve."""
    from oracle.solve import OracleProblem
    _, rep = OracleProblem(sweep_sample_spec(s)).solve()
    return rep.iterations, rep.iterations * (s["n"] + 1) ** 2


def oracle_rate(args, budget_s):
    """The oracle as it stands on this host's cores, on a bounded sample of the
    same workload: returns (it*DOF/s, description, cores, seconds)."""
    from oracle.solve import OracleProblem
    cores = len(os.sched_getaffinity(0))
    if args.workload == "sweep":
        # sample-parallel over all host cores (one sample per process):
        # every 7th sample of the (n, shift strength)-sorted sweep, in a seeded
        # shuffled order; samples still running when the budget ends are dropped
        import multiprocessing as mp
        order = rank_samples(0, 1)[::7]
        np.random.default_rng(0).shuffle(order)
        saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in saved:
            os.environ[k] = "1"
        t0 = time.perf_counter()
        dofs = its = done = 0
        pool = mp.get_context("spawn").Pool(cores)
        try:
            it = pool.imap_unordered(_oracle_sweep_sample, order, chunksize=1)
            while True:
                left = budget_s - (time.perf_counter() - t0)
                if left <= 0:
                    break
                try:
                    a, d = it.next(timeout=left)
                except (StopIteration, mp.TimeoutError):
                    break
                its += a
                dofs += d
                done += 1
        finally:
            dt = time.perf_counter() - t0
            pool.terminate()
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        return dofs / dt, (f"{done} cfg1 samples (every 7th of the (n, shift)-sorted sweep, shuffled) "
                           f"finished in {dt:.1f} s by a pool of {cores} single-threaded processes, "
                           f"setup+factor+solve each, {its} iterations"), cores, dt
    if args.workload == "search":
        from oracle.shift_search import search_sample
        from workloads.configs import search_rhs, search_sample_spec, search_samples
        smp = sorted(search_samples(SEARCH_COUNT, seed=0, levels=SEARCH_LEVELS), key=lambda x: x["n"])
        t0 = time.perf_counter()
        dofs = done = 0
        for x in smp[::max(1, len(smp) // 12)]:
            its = []
            search_sample(search_sample_spec(x), search_rhs(x, seed=0), iters=its)
            dofs += sum(its) * (x["n"] + 1) ** 2
            done += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return dofs / dt, (f"{done} search samples (size-stratified; golden-section, 12 oracle "
                           f"solves each) in {dt:.1f} s"), cores, dt
    spec = config_spec(args.workload)
    t0 = time.perf_counter()
    op = OracleProblem(spec)
    fixed = 4 if spec.n >= 512 else 0
    _, rep = op.solve(fixed_iters=fixed)
    dt = time.perf_counter() - t0
    what = f"fixed {fixed} iterations" if fixed else "full solve"
    return rep.iterations * spec.n_nodes / dt, (f"{args.workload}: setup + coarse LU + {what} "
                                                 f"({rep.iterations} its) in {dt:.1f} s"), cores, dt


PHASE_KERNELS = {"pre": "k_pre2d / k_pre3d (fused 2x Jacobi + residual + I^T restriction)",
                 "coarse": "nd_solve (k_nd_* forward/backward GEMV sweeps of one coarse solve)",
                 "coarse_fd": "fd_solve (k_fd_fold, 2d x k_fd_gemm complex FP64 DMMA GEMMs, k_fd_unfold)",
                 "post": "k_post2d / k_post3d (fused I e_c + 2x Jacobi + A_0 apply)",
                 "krylov": "k_mdot + k_update (CGS multi-dot, update + norm + Givens)"}


def measured_traffic(workload):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of each phase's
    kernels for this workload, from the committed capture summary
    (profiles/r02/traffic.json, written by scripts/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except Exception:
        return None


def roofline(tm, out, args, peak, peak_kind, mma_peak=None):
    """Per-phase HBM rates from the sampled CUDA-event phase timers:
    algorithmic bytes = SURVEY.md 8(d)'s per-step model ("model": every Jacobi
    step, transfer and apply a separate pass), next to our fused kernels'
    compulsory bytes ("fused").  A fast-diagonalisation coarse phase (dense
    complex GEMMs) is tensor-bound: its algorithmic flops / time against the
    measured FP64 MMA peak."""
    phases = {}
    for ph in ("pre", "coarse", "post", "krylov"):
        d = tm[ph]
        if d["ms"] > 0 and d["launches"] > 0:
            sec = d["ms"] * 1e-3
            phases[ph] = {"ms": d["ms"], "launches": int(d["launches"]), "avg_us": 1e3 * d["ms"] / d["launches"],
                          "model_bytes_per_launch": d["model"] / d["launches"],
                          "fused_bytes_per_launch": d["bytes"] / d["launches"],
                          "achieved_gbs": d["model"] / sec / 1e9, "frac": d["model"] / sec / 1e9 / peak,
                          "fused_gbs": d["bytes"] / sec / 1e9, "fused_frac": d["bytes"] / sec / 1e9 / peak}
    if not phases:
        return None
    # dominant phase: the largest share of the serialised ncu time of the same workload
    # (profiles/r02/traffic.json time_share) when committed -- concurrent engine streams
    # time-share the SMs, so live per-launch event times overstate every phase by
    # different factors -- else the largest summed event time
    tr = measured_traffic(args.workload)
    ts = (tr or {}).get("time_share", {})
    if all(ph in ts for ph in phases):
        dom = max(phases, key=lambda k: ts[k])
        dom_by = "ncu serialised time share (profiles/r02/traffic.json): " + \
                 ", ".join(f"{k} {ts[k]:.3f}" for k in phases)
    else:
        dom = max(phases, key=lambda k: phases[k]["ms"])
        dom_by = "largest summed per-launch event time"
    tot_ms = sum(v["ms"] for v in phases.values())
    step_s = out["ms_per_step"] * 1e-3
    for ph, v in phases.items():
        # concurrent sweep streams overlap launches, so per-launch durations overstate
        # each kernel's exclusive cost: also split the step's wall time over the phases
        # in proportion to their summed sampled device time (setup included: a lower bound)
        ba = tm[ph].get("model_all", 0.0) / args.steps
        if ba > 0 and tot_ms > 0:
            v["wall_share_frac"] = ba / (step_s * v["ms"] / tot_ms) / 1e9 / peak
    ball = sum(tm[ph].get("model_all", 0.0) for ph in phases) / args.steps
    fall = sum(tm[ph].get("bytes_all", 0.0) for ph in phases) / args.steps
    agg = {"model_bytes_per_step": ball, "fused_bytes_per_step": fall,
           "frac": ball / step_s / 1e9 / peak, "fused_frac": fall / step_s / 1e9 / peak,
           "note": "bytes of every iteration / whole step time (setup and factorisation included)"}
    fd = tm.get("coarse_flops", 0.0) > 0 and "coarse" in phases
    if fd:
        c = phases["coarse"]
        sec = c["ms"] * 1e-3
        c["bound"] = "tensor"
        c["flops_per_launch"] = tm["coarse_flops"] / c["launches"]
        c["achieved_tflops"] = tm["coarse_flops"] / sec / 1e12
        c["tflops_frac"] = c["achieved_tflops"] / mma_peak if mma_peak else None
        fa = tm.get("coarse_flops_all", 0.0) / args.steps
        if fa > 0 and tot_ms > 0 and mma_peak:
            c["wall_share_tflops_frac"] = fa / (step_s * c["ms"] / tot_ms) / 1e12 / mma_peak
    p = phases[dom]
    if fd and dom == "coarse":
        return {"bound": "tensor", "kernel": PHASE_KERNELS["coarse_fd"], "phase": dom,
                "achieved": p["achieved_tflops"], "peak": mma_peak, "unit": "TFLOP/s",
                "frac": p["tflops_frac"],
                "traffic": (tr or {}).get("coarse_fd", {}).get("dram_bytes_per_launch"),
                "traffic_source": (tr or {}).get("source"),
                "peak_source": "measured (hh_fp64_mma_peak: mma.sync m8n8k4 f64 microbenchmark, this run)",
                "flops_model": "8 real flops per complex multiply-add of the 2d folded transforms: "
                               "2D 128 P^3, 3D 384 P^4 per sample and solve (P = nc/2 + 1); DESIGN.md section 7e",
                "frac_wall_share": p.get("wall_share_tflops_frac"), "dominant_by": dom_by,
                "phases": phases, "aggregate": agg,
                "hbm_peak": peak, "hbm_peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    return {"bound": "hbm", "kernel": PHASE_KERNELS[dom], "phase": dom, "achieved": p["achieved_gbs"],
            "peak": peak, "unit": "GB/s", "frac": p["frac"],
            "traffic": (tr or {}).get(dom, {}).get("dram_bytes_per_launch"),
            "traffic_source": (tr or {}).get("source"),
            "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
            "bytes_model": "SURVEY.md 8(d) per-step model bytes per launch (fused kernels' compulsory "
                           "bytes alongside as fused_*); DESIGN.md section 6",
            "frac_wall_share": p.get("wall_share_frac"), "dominant_by": dom_by, "phases": phases,
            "aggregate": agg}


COARSE = {"auto": 0, "nd": 1, "fd": 3}   # HH_COARSE_AUTO / _ND / _FD (include/hh.h)


def hh_mma_peak(dev):
    """Measured FP64 tensor-core TFLOP/s (after the timed region)."""
    import paper_2104_01439_b200.hh as hh
    return hh.fp64_mma_peak(dev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="sweep", choices=["sweep", "search", "cfg0", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the fresh-process first-call e2e")
    ap.add_argument("--coarse", choices=["replicated", "dist"], default="replicated",
                    help="coarse factor of a slab-decomposed single solve (N > 1)")
    ap.add_argument("--coarse-solver", choices=["auto", "nd", "fd"], default="auto",
                    help="coarse solver (HH_COARSE_AUTO / _ND / _FD)")
    ap.add_argument("--sharding", choices=["roundrobin", "groups"], default="groups",
                    help="sweep samples over ranks (see rank_samples)")
    ap.add_argument("--check-every", type=int, default=1,
                    help="host reads the device convergence flags every this many iterations")
    ap.add_argument("--records", default=None, help="write the sweep's gathered per-sample records (JSONL)")
    ap.add_argument("--cold-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cold_probe:
        run_cold_probe(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # reference arm = the CPU oracle (no installable reference exists)
        if rank != 0:
            return
        # each step a bounded sample, sized so that the whole run ends within minutes
        budget = float(min(20.0, max(5.0, 150.0 / max(1, args.steps + args.warmup))))
        vals = []
        for _ in range(args.warmup):
            oracle_rate(args, budget / 4)
        desc = cores = None
        tot = 0.0
        for _ in range(args.steps):
            v, desc, cores, dt = oracle_rate(args, budget)
            vals.append(v)
            tot += dt
        v = float(np.mean(vals))
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
                "data": "synthetic", "config": {"workload": args.workload, "oracle": "numpy/scipy CPU"},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                 "sample": desc},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(local)
    dev = torch.cuda.current_device()
    out = run_ours(args, rank, world, dev)
    if rank != 0:
        dist.destroy_process_group()
        return
    peak, peak_kind = peaks()
    tm = out["timers"]
    roof = None
    if tm:
        mma_peak = hh_mma_peak(dev) if tm.get("coarse_flops", 0.0) > 0 else None
        roof = roofline(tm, out, args, peak, peak_kind, mma_peak)
    line = {"metric": METRIC, "value": out["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": out["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak" if args.workload == "search" else "strong",
            "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": out["wl"], "e2e": out["e2e"], "roofline": roof,
            "clocks": out["clocks"], "gpu_launches": int(tm["launches"]) if tm else None,
            "iterations_total": out["iterations_total"]}
    if world == 1 and not args.no_cpu_baseline:
        v, desc, cores, _ = oracle_rate(args, 20.0)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": desc}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
