"""Thin ctypes binding of the C ABI in include/hh.h (argument marshalling only).

Every step of the solve runs in libhh.so's CUDA kernels; this module only
checks tensor dtypes/devices/lengths, passes pointers and the current torch
stream, and converts status codes into exceptions.  There is NO CPU fallback:
if libhh.so is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch   # loads libcudart.so.12 into the process before libhh.so

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HH_LIB") or os.path.join(_HERE, "libhh.so")

HH_OP_A0, HH_OP_AEPS, HH_OP_AEPS_COARSE = 0, 1, 2
HH_COARSE_AUTO, HH_COARSE_ND, HH_COARSE_ND_DIST, HH_COARSE_FD = 0, 1, 2, 3
STATUS = {0: "HH_OK", 1: "HH_E_ARG", 2: "HH_E_CONFIG", 3: "HH_E_DIM", 4: "HH_E_CUDA",
          5: "HH_E_NCCL", 6: "HH_E_OOM", 7: "HH_E_SINGULAR", 8: "HH_E_BREAKDOWN",
          9: "HH_E_DIVERGED", 10: "HH_E_STATE"}

EXPORTS = ["hh_setup_problem", "hh_layout", "hh_local_layout", "hh_apply_op", "hh_vcycle",
           "hh_coarse_solve", "hh_fgmres_solve", "hh_fgmres_solve_host", "hh_sweep",
           "hh_destroy_problem", "hh_reset_timers", "hh_read_timers", "hh_sweep_timers",
           "hh_slab_bounds", "hh_nccl_unique_id", "hh_shift_search", "hh_lfa_rho", "hh_lfa_sigma_c", "hh_lfa_stats",
           "hh_arnoldi_orthogonality", "hh_fp64_peak", "hh_coarse_flops", "hh_coarse_kind", "hh_fp64_mma_peak", "hh_last_error", "hh_version"]


class ProblemDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n_cells", C.c_int32), ("k_const", C.c_double),
                ("k_elem", C.POINTER(C.c_double)), ("k_elem_coarse", C.POINTER(C.c_double)),
                ("beta", C.c_double), ("sigma", C.c_double), ("nu_pre", C.c_int32),
                ("nu_post", C.c_int32), ("omega", C.c_double), ("coarse_solver", C.c_int32),
                ("device", C.c_int32), ("stream", C.c_void_p), ("max_restart", C.c_int32),
                ("nslabs_local", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_id", C.c_void_p), ("shift_map", C.c_int32)]


class FgmresOpts(C.Structure):
    _fields_ = [("restart", C.c_int32), ("max_iters", C.c_int32), ("fixed_iters", C.c_int32),
                ("rtol", C.c_double), ("check_every", C.c_int32), ("reorth", C.c_int32)]


class FgmresReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("restarts", C.c_int32), ("converged", C.c_int32),
                ("rel_res_lsq", C.c_double), ("rel_res_true", C.c_double), ("rho", C.c_double),
                ("setup_s", C.c_double), ("solve_s", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Sample(C.Structure):
    _fields_ = [("id", C.c_int64), ("n_cells", C.c_int32), ("k", C.c_double),
                ("beta", C.c_double), ("sigma", C.c_double)]


class SearchSample(C.Structure):
    _fields_ = [("id", C.c_int64), ("n_cells", C.c_int32), ("k", C.c_double), ("beta", C.c_double)]


class LfaQuery(C.Structure):
    _fields_ = [("k", C.c_double), ("h", C.c_double), ("beta", C.c_double), ("sigma", C.c_double),
                ("omega", C.c_double), ("nu1", C.c_int32), ("nu2", C.c_int32), ("m", C.c_int32),
                ("pad", C.c_int32)]


class SearchResult(C.Structure):
    _fields_ = [("id", C.c_int64), ("status", C.c_int32), ("evaluations", C.c_int32),
                ("iterations_total", C.c_int32), ("sigma_hat", C.c_double),
                ("sigma_best", C.c_double), ("rho_best", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SampleResult(C.Structure):
    _fields_ = [("id", C.c_int64), ("status", C.c_int32), ("iterations", C.c_int32),
                ("converged", C.c_int32), ("rel_res_true", C.c_double), ("rho", C.c_double),
                ("setup_s", C.c_double), ("solve_s", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class HHError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhh.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    vp, i32, dp = C.c_void_p, C.c_int32, C.POINTER(C.c_double)
    sigs = {
        "hh_setup_problem": [C.POINTER(ProblemDesc), C.POINTER(vp)],
        "hh_layout": [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
        "hh_local_layout": [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
        "hh_slab_bounds": [i32, i32, C.POINTER(C.c_int32)],
        "hh_nccl_unique_id": [vp],
        "hh_shift_search": [C.POINTER(ProblemDesc), C.POINTER(FgmresOpts), C.POINTER(SearchSample), i32,
                            C.POINTER(C.c_void_p), C.c_double, C.c_double, C.c_double,
                            C.POINTER(SearchResult)],
        "hh_lfa_rho": [C.POINTER(LfaQuery), i32, i32, dp],
        "hh_lfa_sigma_c": [C.POINTER(LfaQuery), i32, i32, C.c_double, C.c_double, C.c_double, dp],
        "hh_lfa_stats": [i32, dp],
        "hh_apply_op": [vp, i32, vp, vp],
        "hh_vcycle": [vp, vp, vp],
        "hh_coarse_solve": [vp, vp, vp],
        "hh_fgmres_solve": [vp, vp, vp, C.POINTER(FgmresOpts), C.POINTER(FgmresReport), dp],
        "hh_fgmres_solve_host": [vp, vp, vp, C.POINTER(FgmresOpts), C.POINTER(FgmresReport)],
        "hh_sweep": [C.POINTER(ProblemDesc), C.POINTER(FgmresOpts), C.POINTER(Sample), i32,
                     C.POINTER(SampleResult)],
        "hh_destroy_problem": [vp],
        "hh_arnoldi_orthogonality": [vp, dp, C.POINTER(C.c_int32)],
        "hh_fp64_peak": [i32, dp, dp],
        "hh_reset_timers": [vp, i32],
        "hh_read_timers": [vp, dp, C.POINTER(C.c_int64)],
        "hh_sweep_timers": [i32, dp, C.POINTER(C.c_int64)],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.hh_last_error.restype = C.c_char_p
    lib.hh_version.restype = C.c_char_p
    return lib


lib = _load()


def _check(st):
    if st != 0:
        raise HHError(st, lib.hh_last_error().decode())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream) if torch.cuda.is_available() else None


def _ptr(t: torch.Tensor, n: int, name: str):
    if not isinstance(t, torch.Tensor) or t.dtype != torch.complex128 or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA complex128 tensor")
    if not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name} must be contiguous with {n} entries (got {t.numel()})")
    return C.c_void_p(t.data_ptr())


def opts(restart=100, max_iters=500, fixed_iters=0, rtol=1e-6, check_every=1, reorth=0):
    """hh_fgmres_opts; reorth: 0 single-pass CGS, 1 selective (DGKS), 2 always (C11)."""
    return FgmresOpts(restart, max_iters, fixed_iters, rtol, check_every, reorth)


class Problem:
    """Owns one hh_problem handle (setup_problem ... destroy_problem)."""

    def __init__(self, dim, n_cells, k_const=0.0, k_elem=None, k_elem_coarse=None, beta=1.0,
                 sigma=1.5, nu_pre=2, nu_post=2, omega=0.6, max_restart=100, device=None,
                 nslabs_local=1, rank=0, nranks=1, nccl_id: bytes | None = None, shift_map=0,
                 coarse_solver=HH_COARSE_AUTO):
        """nslabs_local > 1: the solve is cut into that many slabs held by this
        process; nccl_id (from nccl_unique_id(), shared by all ranks): this
        process holds slab `rank` of `nranks` (one GPU per process).  Vectors
        then hold this handle's owned planes (local_layout()).  coarse_solver =
        HH_COARSE_ND_DIST distributes the coarse factor over the slabs; HH_COARSE_FD
        solves it by fast diagonalisation (constant k); AUTO picks FD for
        constant k where it pays and the ND factor otherwise."""
        self.handle = C.c_void_p()
        dev = torch.cuda.current_device() if device is None else device
        d = ProblemDesc()
        d.dim, d.n_cells, d.k_const = dim, n_cells, float(k_const)
        keep = []
        if k_elem is not None:
            kf = np.ascontiguousarray(k_elem, dtype=np.float64)
            kc = np.ascontiguousarray(k_elem_coarse, dtype=np.float64)
            if kf.size != n_cells ** dim or kc.size != (n_cells // 2) ** dim:
                raise ValueError("k_elem / k_elem_coarse have the wrong size")
            keep = [kf, kc]
            d.k_elem = kf.ctypes.data_as(C.POINTER(C.c_double))
            d.k_elem_coarse = kc.ctypes.data_as(C.POINTER(C.c_double))
        d.beta, d.sigma, d.nu_pre, d.nu_post, d.omega = beta, sigma, nu_pre, nu_post, omega
        d.coarse_solver = coarse_solver
        d.device = dev
        d.stream = _stream()
        d.max_restart = max_restart
        d.nslabs_local, d.rank, d.nranks = nslabs_local, rank, nranks
        d.shift_map = shift_map
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be 128 bytes")
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = C.cast(idbuf, C.c_void_p)
        with torch.cuda.device(dev):
            _check(lib.hh_setup_problem(C.byref(d), C.byref(self.handle)))
        del keep, idbuf
        nf, nc = C.c_int64(), C.c_int64()
        _check(lib.hh_layout(self.handle, C.byref(nf), C.byref(nc)))
        self.n_fine, self.n_coarse = nf.value, nc.value
        self.dim, self.n_cells, self.device = dim, n_cells, dev

    def coarse_kind(self):
        """hh_coarse_kind: the coarse solver in use (HH_COARSE_ND / _ND_DIST / _FD)."""
        k = C.c_int32()
        _check(lib.hh_coarse_kind(self.handle, C.byref(k)))
        return k.value

    def local_layout(self):
        """(n_local_nodes, first_plane, n_planes) of the owned slab range."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.hh_local_layout(self.handle, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @classmethod
    def from_spec(cls, spec, max_restart=None, **kw):
        """Build from a workloads.ProblemSpec (inputs only)."""
        kw.setdefault("shift_map", getattr(spec, "shift_map", 0))
        return cls(spec.dim, spec.n, k_const=spec.k_const or 0.0, k_elem=spec.k_fine,
                   k_elem_coarse=spec.k_coarse, beta=spec.beta, sigma=spec.sigma,
                   nu_pre=spec.nu_pre, nu_post=spec.nu_post, omega=spec.omega,
                   max_restart=max_restart or spec.restart, **kw)

    def new_vector(self, coarse=False):
        return torch.zeros(self.n_coarse if coarse else self.n_fine, dtype=torch.complex128,
                           device=f"cuda:{self.device}")

    def apply_op(self, op, x, y=None):
        n = self.n_coarse if op == HH_OP_AEPS_COARSE else self.n_fine
        y = self.new_vector(op == HH_OP_AEPS_COARSE) if y is None else y
        _check(lib.hh_apply_op(self.handle, op, _ptr(x, n, "x"), _ptr(y, n, "y")))
        return y

    def vcycle(self, f, z=None):
        z = self.new_vector() if z is None else z
        _check(lib.hh_vcycle(self.handle, _ptr(f, self.n_fine, "f"), _ptr(z, self.n_fine, "z")))
        return z

    def coarse_solve(self, r, e=None):
        e = self.new_vector(True) if e is None else e
        _check(lib.hh_coarse_solve(self.handle, _ptr(r, self.n_coarse, "r"),
                                   _ptr(e, self.n_coarse, "e")))
        return e

    def fgmres_solve(self, b, x=None, o=None, history=False):
        """x: the initial guess x0 on entry (zeros if None), the solution on exit."""
        x = self.new_vector() if x is None else x
        o = o or opts()
        rep = FgmresReport()
        hist = (C.c_double * (max(o.max_iters, o.fixed_iters) + 2))() if history else None
        _check(lib.hh_fgmres_solve(self.handle, _ptr(b, self.n_fine, "b"), _ptr(x, self.n_fine, "x"),
                                   C.byref(o), C.byref(rep), hist))
        out = rep.as_dict()
        if history:
            out["history"] = list(hist[: rep.iterations + 1])
        return x, out

    def fgmres_solve_host(self, b_host: np.ndarray, x_host: np.ndarray, o=None):
        """End-to-end call with HOST complex128 arrays (pinned or pageable)."""
        o = o or opts()
        rep = FgmresReport()
        assert b_host.dtype == np.complex128 and x_host.dtype == np.complex128
        _check(lib.hh_fgmres_solve_host(self.handle, C.c_void_p(b_host.ctypes.data),
                                        C.c_void_p(x_host.ctypes.data), C.byref(o), C.byref(rep)))
        return rep.as_dict()

    def arnoldi_orthogonality(self):
        """(max |<v_a, v_c> - delta_ac|, number of basis vectors) of the last Arnoldi cycle."""
        loss, nv = C.c_double(), C.c_int32()
        _check(lib.hh_arnoldi_orthogonality(self.handle, C.byref(loss), C.byref(nv)))
        return loss.value, nv.value

    def reset_timers(self, enable=True):
        _check(lib.hh_reset_timers(self.handle, int(enable)))

    def read_timers(self):
        st = (C.c_double * 24)()
        nl = C.c_int64()
        _check(lib.hh_read_timers(self.handle, st, C.byref(nl)))
        return _phase_dict(st, nl.value)

    def close(self):
        if self.handle:
            lib.hh_destroy_problem(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sweep(samples, nu_pre=2, nu_post=2, omega=0.6, o=None, device=None, max_restart=100,
          coarse_solver=HH_COARSE_AUTO):
    """hh_sweep over a list of dicts with keys id, n, k, beta, sigma."""
    o = o or opts()
    d = ProblemDesc()
    d.dim, d.nu_pre, d.nu_post, d.omega = 2, nu_pre, nu_post, omega
    d.device = torch.cuda.current_device() if device is None else device
    d.stream = _stream()
    d.max_restart = max_restart
    d.coarse_solver = coarse_solver
    n = len(samples)
    arr = (Sample * n)(*[Sample(s["id"], s["n"], s["k"], s["beta"], s["sigma"]) for s in samples])
    out = (SampleResult * n)()
    _check(lib.hh_sweep(C.byref(d), C.byref(o), arr, n, out))
    return [r.as_dict() for r in out]


def shift_search(samples, rhs, lo=1.0, hi=2.0, tol=1e-2, o=None, nu_pre=2, nu_post=2, omega=0.6,
                 device=None, max_restart=100, coarse_solver=HH_COARSE_AUTO):
    """hh_shift_search: golden-section sigma search per sample (dicts with id, n, k,
    beta); rhs[i] = host complex128 right-hand side of sample i (reused for all sigma).
    Default budget = the paper's: rtol 1e-8, 50 iterations, no restart."""
    o = o or opts(restart=50, max_iters=50, rtol=1e-8)
    d = ProblemDesc()
    d.dim, d.nu_pre, d.nu_post, d.omega = 2, nu_pre, nu_post, omega
    d.device = torch.cuda.current_device() if device is None else device
    d.stream = _stream()
    d.max_restart = max_restart
    d.coarse_solver = coarse_solver
    n = len(samples)
    arr = (SearchSample * n)(*[SearchSample(s["id"], s["n"], s["k"], s.get("beta", 1.0)) for s in samples])
    keep = [np.ascontiguousarray(r, dtype=np.complex128) for r in rhs]
    for s_, r in zip(samples, keep):
        if r.size != (s_["n"] + 1) ** 2:
            raise ValueError("rhs size mismatch")
    ptrs = (C.c_void_p * n)(*[r.ctypes.data for r in keep])
    out = (SearchResult * n)()
    _check(lib.hh_shift_search(C.byref(d), C.byref(o), arr, n, ptrs, lo, hi, tol, out))
    del keep
    return [r.as_dict() for r in out]


def _lfa_queries(queries):
    return (LfaQuery * len(queries))(*[LfaQuery(q["k"], q["h"], q.get("beta", 1.0), q.get("sigma", 1.0),
                                                q.get("omega", 0.6), q.get("nu1", 2), q.get("nu2", 2),
                                                q.get("m", 128), 0) for q in queries])


def lfa_rho(queries, device=None):
    """hh_lfa_rho: rho_loc of the two-grid symbol for dicts with
    k, h, beta, sigma, omega, nu1, nu2, m (theta grid m x m of T^low)."""
    n = len(queries)
    out = (C.c_double * n)()
    dev = torch.cuda.current_device() if device is None else device
    _check(lib.hh_lfa_rho(_lfa_queries(queries), n, dev, out))
    return list(out)


def lfa_sigma_c(queries, lo=1.0, hi=2.0, tol=1e-3, device=None):
    """hh_lfa_sigma_c: smallest sigma in [lo, hi] with rho_loc < 1
    by bisection to width tol; NaN when rho_loc(hi) >= 1."""
    n = len(queries)
    out = (C.c_double * n)()
    dev = torch.cuda.current_device() if device is None else device
    _check(lib.hh_lfa_sigma_c(_lfa_queries(queries), n, dev, lo, hi, tol, out))
    return list(out)


def lfa_stats(reset=False):
    """hh_lfa_stats: theta evaluations, Aberth iterations, kernel ms, launches."""
    st = (C.c_double * 4)()
    _check(lib.hh_lfa_stats(1 if reset else 0, st))
    return {"evals": st[0], "aberth_iters": st[1], "ms": st[2], "launches": int(st[3])}


PHASES = ("pre", "coarse", "post", "krylov")


def _phase_dict(st, launches):
    d = {"launches": launches}
    for i, ph in enumerate(PHASES):
        d[ph] = {"ms": st[i], "bytes": st[4 + i], "launches": st[8 + i], "bytes_all": st[12 + i],
                 "model": st[16 + i], "model_all": st[20 + i]}
    return d


def sweep_timers(reset_enable=-1):
    st = (C.c_double * 24)()
    nl = C.c_int64()
    _check(lib.hh_sweep_timers(reset_enable, st, C.byref(nl)))
    return _phase_dict(st, nl.value)


def coarse_flops(problem=None):
    """hh_coarse_flops: (timed, all) coarse-solve flops since the last timer reset
    of `problem` (a Problem) or, with None, of the sweep."""
    out = (C.c_double * 2)()
    _check(lib.hh_coarse_flops(problem.handle if problem is not None else None, out))
    return out[0], out[1]


def fp64_peak(device=None):
    """(measured FP64 TFLOP/s, nominal SM MHz) from the DFMA microbenchmark."""
    t, mhz = C.c_double(), C.c_double()
    dev = torch.cuda.current_device() if device is None else device
    _check(lib.hh_fp64_peak(dev, C.byref(t), C.byref(mhz)))
    return t.value, mhz.value


def fp64_mma_peak(device=None):
    """Measured FP64 tensor-core (mma.sync m8n8k4 f64) TFLOP/s."""
    t = C.c_double()
    dev = torch.cuda.current_device() if device is None else device
    _check(lib.hh_fp64_mma_peak(dev, C.byref(t)))
    return t.value


def version():
    return lib.hh_version().decode()


def slab_bounds(n_cells, nslabs):
    """Plane bounds z[0..nslabs] of the slab decomposition (slab k owns [z[k], z[k+1]))."""
    z = (C.c_int32 * (nslabs + 1))()
    _check(lib.hh_slab_bounds(n_cells, nslabs, z))
    return list(z)


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (call on one rank, broadcast to the others)."""
    buf = C.create_string_buffer(128)
    _check(lib.hh_nccl_unique_id(buf))
    return buf.raw
