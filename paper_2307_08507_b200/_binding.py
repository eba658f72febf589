"""ctypes marshalling for include/mdot.h (no computation happens here)."""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MDOT_LIB: load another build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("MDOT_LIB") or os.path.join(_HERE, "libmdot_b200.so")

MDOT_COST_DENSE_F32, MDOT_COST_SQEUCLID_F32, MDOT_COST_DENSE_F64, MDOT_COST_SQEUCLID_DOT_F32 = 0, 1, 2, 3
MDOT_MEM_HOST, MDOT_MEM_DEVICE = 0, 1
MDOT_SCHED_FIXED, MDOT_SCHED_DOUBLING, MDOT_SCHED_EXPLICIT, MDOT_SCHED_ADAPTIVE = 0, 1, 2, 3
MDOT_PROJ_PNCG, MDOT_PROJ_SINKHORN, MDOT_PROJ_NCG, MDOT_PROJ_PNCG_JACOBI = 0, 1, 2, 3
MDOT_BETA_PPR, MDOT_BETA_PPR_AF, MDOT_BETA_PFR, MDOT_BETA_PPR_PLUS = 0, 1, 2, 3
MDOT_WARM_SCALED, MDOT_WARM_CARRY, MDOT_WARM_ZERO = 0, 1, 2
MDOT_PREC_AUTO, MDOT_PREC_F32P, MDOT_PREC_F64P = 0, 1, 2
STATUS_NAMES = {0: "MDOT_OK", 1: "MDOT_EINVAL", 2: "MDOT_EGEN", 3: "MDOT_EINSTABLE",
                4: "MDOT_ENOCONV", 5: "MDOT_ELINESEARCH", 6: "MDOT_ECUDA", 7: "MDOT_ENCCL",
                8: "MDOT_ENOMEM"}


class MdotError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Problem(ct.Structure):
    _fields_ = [("n", ct.c_int64), ("kind", ct.c_int32), ("mem", ct.c_int32),
                ("C", ct.c_void_p), ("d", ct.c_int32), ("scale", ct.c_float),
                ("X", ct.c_void_p), ("Y", ct.c_void_p), ("r", ct.c_void_p), ("c", ct.c_void_p)]


class Schedule(ct.Structure):
    _fields_ = [("kind", ct.c_int32), ("T", ct.c_int32), ("gamma_bar", ct.c_double),
                ("step_max", ct.c_double), ("gamma0", ct.c_double), ("gammas", ct.c_void_p),
                ("n_gammas", ct.c_int32)]


class TraceRec(ct.Structure):
    """mdot_trace_rec (include/mdot.h): one PNCG iteration / Sinkhorn half-step."""
    _fields_ = [("t", ct.c_int32), ("k", ct.c_int32), ("l1", ct.c_double), ("rho", ct.c_double),
                ("alpha", ct.c_double), ("dphi0", ct.c_double), ("dphi_alpha", ct.c_double),
                ("dphi_value", ct.c_double), ("trials", ct.c_int32), ("reset", ct.c_int32),
                ("beta", ct.c_double), ("gs", ct.c_double)]


class Options(ct.Structure):
    _fields_ = [("eps", ct.c_double), ("stop", ct.c_int32), ("projector", ct.c_int32),
                ("beta", ct.c_int32), ("c1", ct.c_double), ("c2", ct.c_double),
                ("warm", ct.c_int32), ("precision", ct.c_int32), ("p0_ones", ct.c_int32),
                ("ls_max_trials", ct.c_int32), ("max_evals", ct.c_int64),
                ("time_kernels", ct.c_int32), ("device_control", ct.c_int32),
                ("stream", ct.c_void_p), ("eps_md", ct.c_double),
                ("trace", ct.c_void_p), ("trace_cap", ct.c_int64), ("trace_len", ct.c_void_p)]


class Result(ct.Structure):
    _fields_ = [("cost_rounded", ct.c_double), ("cost_unrounded", ct.c_double),
                ("l1_final", ct.c_double), ("rho_final", ct.c_double), ("gamma_bar", ct.c_double),
                ("seconds", ct.c_double), ("kernel_ms", ct.c_double),
                ("md_steps", ct.c_int64), ("iterations", ct.c_int64), ("evaluations", ct.c_int64),
                ("ls_evaluations", ct.c_int64), ("resets", ct.c_int64), ("ls_restarts", ct.c_int64),
                ("fallbacks", ct.c_int64), ("kernel_launches", ct.c_int64), ("all_launches", ct.c_int64),
                ("stage_ms", ct.c_double * 4), ("stage_samples", ct.c_int64),
                ("status", ct.c_int32), ("control_path", ct.c_int32),
                ("rho0", ct.c_double * 64), ("l10", ct.c_double * 64),
                ("iters_step", ct.c_int64 * 64), ("gammas", ct.c_double * 64)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_
             if f not in ("rho0", "l10", "iters_step", "stage_ms", "gammas")}
        d["stage_ms"] = list(self.stage_ms)
        T = int(min(self.md_steps, 64))
        d["rho0"] = list(self.rho0)[:T]
        d["l10"] = list(self.l10)[:T]
        d["iters_step"] = list(self.iters_step)[:T]
        d["gammas"] = list(self.gammas)[:T]
        d["status_name"] = STATUS_NAMES.get(self.status, str(self.status))
        return d


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2307_08507_b200/build.py "
                              "(there is no CPU fallback)")
        L = ct.CDLL(LIB_PATH)
        P = ct.c_void_p
        D = ct.c_double
        L.mdot_last_error.restype = ct.c_char_p
        L.mdot_abi_version.restype = ct.c_int32
        L.mdot_options_default.argtypes = [ct.POINTER(Options)]
        L.mdot_schedule_default.argtypes = [ct.POINTER(Schedule)]
        sig_solve = [ct.POINTER(Problem), ct.POINTER(Schedule), ct.POINTER(Options), P, P, P,
                     ct.POINTER(Result)]
        for nm in ("mdot_solve", "mdot_sinkhorn"):
            getattr(L, nm).argtypes = sig_solve
            getattr(L, nm).restype = ct.c_int
        L.mdot_solve_batch.argtypes = [ct.POINTER(Problem), ct.c_int32, P, P, ct.POINTER(Schedule),
                                       ct.POINTER(Options), P, P, ct.POINTER(Result)]
        L.mdot_marginals.argtypes = [ct.POINTER(Problem), P, P, D, P, P, ct.POINTER(Options),
                                     ct.POINTER(ct.c_int32)]
        L.mdot_round.argtypes = [ct.POINTER(Problem), P, P, D, P, ct.POINTER(D), ct.POINTER(D),
                                 ct.POINTER(Options)]
        L.mdot_get_unique_id.argtypes = [P]
        L.mdot_comm_create.argtypes = [P, ct.c_int32, ct.c_int32, ct.c_int32, ct.POINTER(P)]
        L.mdot_comm_destroy.argtypes = [P]
        L.mdot_comm_create_local.argtypes = [ct.c_char_p, ct.c_int32, ct.c_int32, ct.c_int32, ct.POINTER(P)]
        L.mdot_comm_enable_peer.argtypes = [P, ct.c_int64]
        L.mdot_solve_sharded.argtypes = [P, ct.POINTER(Problem), ct.c_int64, ct.c_int64,
                                         ct.POINTER(Schedule), ct.POINTER(Options), P, P,
                                         ct.POINTER(Result)]
        if hasattr(L, "mdot_solve_sharded_2d"):   # absent from libraries built before session 4 (A/B builds)
            L.mdot_solve_sharded_2d.argtypes = [P, P, ct.POINTER(Problem), ct.c_int64, ct.c_int64, ct.c_int64,
                                                ct.c_int64, ct.POINTER(Schedule), ct.POINTER(Options), P, P,
                                                ct.POINTER(Result)]
            L.mdot_solve_sharded_2d.restype = ct.c_int
        if hasattr(L, "mdot_last_screen_stats"):   # absent from libraries built before K2s (A/B builds)
            L.mdot_last_screen_stats.argtypes = [ct.POINTER(D)]
            L.mdot_last_screen_stats.restype = ct.c_int
        for nm in ("mdot_solve_batch", "mdot_marginals", "mdot_round", "mdot_get_unique_id",
                   "mdot_comm_create", "mdot_comm_create_local", "mdot_comm_enable_peer", "mdot_comm_destroy",
                   "mdot_solve_sharded"):
            getattr(L, nm).restype = ct.c_int
        if L.mdot_abi_version() != 3:
            raise ImportError("libmdot_b200.so ABI version mismatch")
        _lib = L
    return _lib


def mdot_last_error() -> str:
    return lib().mdot_last_error().decode()


def mdot_last_screen_stats() -> dict:
    """K2s statistics of this thread's last solve (include/mdot.h)."""
    out = (ct.c_double * 5)()
    lib().mdot_last_screen_stats(out)
    return {"kept": out[0], "screened": out[1], "evals": int(out[2]), "ms": out[3], "timed": int(out[4]),
            "kept_frac": (out[0] / out[1]) if out[1] else None}


# ---------------------------------------------------------------- marshalling
def _is_cuda(x):
    return hasattr(x, "is_cuda") and x.is_cuda


F64, F32 = ("float64",), ("float32",)
F32_OR_F64 = ("float32", "float64")


def _dtname(x):
    return str(x.dtype).replace("torch.", "") if hasattr(x, "data_ptr") else np.dtype(x.dtype).name


def _check_arr(name, x, dtypes, cuda=None):
    """The C side reads / writes these buffers with a fixed element type
    (include/mdot.h): a float32 buffer passed where fp64 is expected would be
    over-read or overwritten by 2x its size.  Also every buffer of one call
    must live where the problem's `mem` kind says."""
    if x is None:
        return
    dt = _dtname(x)
    if dt not in dtypes:
        raise TypeError(f"{name}: dtype {dt}, expected {' or '.join(dtypes)}")
    if cuda is not None and _is_cuda(x) != cuda:
        raise TypeError(f"{name}: {'host' if cuda else 'device'} buffer expected (same memory kind as the problem)")


def _ptr(x, dtypes=None, name="array", cuda=None):
    """Raw pointer of a contiguous torch tensor / numpy array (None -> NULL);
    with `dtypes`, the element type (and memory kind) is checked first."""
    if x is None:
        return None
    if dtypes is not None:
        _check_arr(name, x, dtypes, cuda)
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ct.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data_as(ct.c_void_p)
    raise TypeError(f"unsupported array type {type(x)}")


def _current_stream():
    import torch
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def problem(C=None, r=None, c=None, *, X=None, Y=None, scale=0.0, n=None, recipe="diff"):
    """Build an mdot_problem; keeps references to the arrays on the struct.
    recipe selects the on-the-fly cost's fp32 op sequence: "diff" (Z22,
    MDOT_COST_SQEUCLID_F32) or "dot" (Z22b, MDOT_COST_SQEUCLID_DOT_F32)."""
    ref = C if C is not None else X
    dev = _is_cuda(ref)
    if C is not None:
        kind = MDOT_COST_DENSE_F64 if str(C.dtype).endswith("float64") else MDOT_COST_DENSE_F32
        nn = C.shape[0] if n is None else n
        d = 0
    else:
        if recipe not in ("diff", "dot"):
            raise ValueError(f"recipe {recipe!r}: 'diff' or 'dot'")
        kind = MDOT_COST_SQEUCLID_DOT_F32 if recipe == "dot" else MDOT_COST_SQEUCLID_F32
        nn = Y.shape[0] if n is None else n
        d = X.shape[1]
    pb = Problem(nn, kind, MDOT_MEM_DEVICE if dev else MDOT_MEM_HOST, _ptr(C, F32_OR_F64, "C", dev), d,
                 float(scale), _ptr(X, F32, "X", dev), _ptr(Y, F32, "Y", dev), _ptr(r, F64, "r", dev),
                 _ptr(c, F64, "c", dev))
    pb._keep = (C, r, c, X, Y)
    return pb


def schedule(kind=MDOT_SCHED_FIXED, gamma_bar=4096.0, T=0, step_max=256.0, gamma0=1.0, gammas=None):
    s = Schedule()
    lib().mdot_schedule_default(ct.byref(s))
    s.kind, s.gamma_bar, s.T, s.step_max, s.gamma0 = kind, float(gamma_bar), int(T), float(step_max), float(gamma0)
    if gammas is not None:
        g = np.ascontiguousarray(gammas, dtype=np.float64)
        s.kind = MDOT_SCHED_EXPLICIT
        s.gammas = g.ctypes.data_as(ct.c_void_p)
        s.n_gammas = len(g)
        s._keep = g
    return s


def options(trace_cap=0, **kw):
    """mdot_options with defaults; trace_cap > 0 attaches a host trace buffer
    (read it back with read_trace(options) after the call)."""
    o = Options()
    lib().mdot_options_default(ct.byref(o))
    for k, v in kw.items():
        if k == "stream":
            continue
        setattr(o, k, v)
    if trace_cap:
        buf = (TraceRec * int(trace_cap))()
        ln = ct.c_int64(0)
        o.trace = ct.cast(buf, ct.c_void_p)
        o.trace_cap = int(trace_cap)
        o.trace_len = ct.cast(ct.pointer(ln), ct.c_void_p)
        o._trace = (buf, ln)
    return o


def read_trace(opts):
    """The records the last call wrote into opts' trace buffer, as dicts."""
    buf, ln = opts._trace
    return [{f: getattr(buf[k], f) for f, _ in TraceRec._fields_} for k in range(ln.value)]


def _check(st, what):
    if st != 0:
        raise MdotError(st, f"{what}: {mdot_last_error()}")


def _solve(fn, C, r, c, X, Y, scale, sched, opts, u_out, v_out, P_out, check, recipe="diff"):
    pb = problem(C, r, c, X=X, Y=Y, scale=scale, recipe=recipe)
    sched = sched if sched is not None else schedule()
    opts = opts if opts is not None else options()
    if pb.mem == MDOT_MEM_DEVICE:
        opts.stream = _current_stream()
    res = Result()
    dev = pb.mem == MDOT_MEM_DEVICE
    st = fn(ct.byref(pb), ct.byref(sched), ct.byref(opts), _ptr(u_out, F64, "u_out", dev),
            _ptr(v_out, F64, "v_out", dev), _ptr(P_out, F32, "P_out", dev), ct.byref(res))
    d = res.as_dict()
    d["status"] = st
    if check and st not in (0,):
        _check(st, fn.__name__)
    return d


def mdot_solve(C=None, r=None, c=None, *, X=None, Y=None, scale=0.0, schedule=None, options=None,
               u_out=None, v_out=None, P_out=None, check=True, recipe="diff"):
    """MDOT-PNCG solve; returns the mdot_result as a dict."""
    return _solve(lib().mdot_solve, C, r, c, X, Y, scale, schedule, options, u_out, v_out, P_out, check, recipe)


def mdot_sinkhorn(C=None, r=None, c=None, *, X=None, Y=None, scale=0.0, schedule=None, options=None,
                  u_out=None, v_out=None, P_out=None, check=True, recipe="diff"):
    """Same solve with Sinkhorn projections (Alg. 3) on the same kernels."""
    return _solve(lib().mdot_sinkhorn, C, r, c, X, Y, scale, schedule, options, u_out, v_out, P_out, check, recipe)


def mdot_solve_batch(C, R, Cm, *, schedule=None, options=None, u_out=None, v_out=None, check=True):
    B, n = R.shape
    pb = problem(C, R[0], Cm[0])
    sched = schedule if schedule is not None else globals()["schedule"]()
    opts = options if options is not None else globals()["options"]()
    if pb.mem == MDOT_MEM_DEVICE:
        opts.stream = _current_stream()
    res = (Result * B)()
    dev = pb.mem == MDOT_MEM_DEVICE
    st = lib().mdot_solve_batch(ct.byref(pb), B, _ptr(R, F64, "R", dev), _ptr(Cm, F64, "Cm", dev), ct.byref(sched),
                                ct.byref(opts), _ptr(u_out, F64, "u_out", dev), _ptr(v_out, F64, "v_out", dev), res)
    if check:
        _check(st, "mdot_solve_batch")
    return [res[b].as_dict() for b in range(B)]


def mdot_marginals(A, B, gbar, C=None, r=None, c=None, *, X=None, Y=None, scale=0.0, lr=None, lc=None,
                   options=None, check=True, recipe="diff"):
    """One fused evaluation: (log r(P), log c(P)) for P = exp(A + B - gbar C)."""
    pb = problem(C, r, c, X=X, Y=Y, scale=scale, recipe=recipe)
    opts = options if options is not None else globals()["options"]()
    if pb.mem == MDOT_MEM_DEVICE:
        import torch
        opts.stream = _current_stream()
        lr = torch.empty(pb.n, dtype=torch.float64, device=A.device) if lr is None else lr
        lc = torch.empty(pb.n, dtype=torch.float64, device=A.device) if lc is None else lc
    else:
        lr = np.empty(pb.n) if lr is None else lr
        lc = np.empty(pb.n) if lc is None else lc
    fb = ct.c_int32(0)
    dev = pb.mem == MDOT_MEM_DEVICE
    st = lib().mdot_marginals(ct.byref(pb), _ptr(A, F64, "A", dev), _ptr(B, F64, "B", dev), float(gbar),
                              _ptr(lr, F64, "lr", dev), _ptr(lc, F64, "lc", dev), ct.byref(opts), ct.byref(fb))
    if check:
        _check(st, "mdot_marginals")
    return lr, lc, int(fb.value)


def mdot_round(U, V, gbar, C=None, r=None, c=None, *, X=None, Y=None, scale=0.0, P_out=None,
               options=None, check=True, recipe="diff"):
    pb = problem(C, r, c, X=X, Y=Y, scale=scale, recipe=recipe)
    opts = options if options is not None else globals()["options"]()
    if pb.mem == MDOT_MEM_DEVICE:
        opts.stream = _current_stream()
    cF = ct.c_double(0)
    cG = ct.c_double(0)
    dev = pb.mem == MDOT_MEM_DEVICE
    st = lib().mdot_round(ct.byref(pb), _ptr(U, F64, "U", dev), _ptr(V, F64, "V", dev), float(gbar),
                          _ptr(P_out, F32, "P_out", dev), ct.byref(cF), ct.byref(cG), ct.byref(opts))
    if check:
        _check(st, "mdot_round")
    return cF.value, cG.value


def mdot_get_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(lib().mdot_get_unique_id(buf), "mdot_get_unique_id")
    return buf.raw


def mdot_comm_create(unique_id: bytes, nranks: int, rank: int, device: int):
    buf = ct.create_string_buffer(bytes(unique_id), 128)
    out = ct.c_void_p()
    _check(lib().mdot_comm_create(buf, nranks, rank, device, ct.byref(out)), "mdot_comm_create")
    return out


def mdot_comm_create_local(group: str, nranks: int, rank: int, device: int):
    out = ct.c_void_p()
    _check(lib().mdot_comm_create_local(group.encode(), nranks, rank, device, ct.byref(out)),
           "mdot_comm_create_local")
    return out


def mdot_comm_enable_peer(comm, n_max: int, check=True):
    """Collective: fused peer exchange for sharded solves with n <= n_max
    (include/mdot.h).  Returns the status when check=False."""
    st = lib().mdot_comm_enable_peer(comm, int(n_max))
    if check:
        _check(st, "mdot_comm_enable_peer")
    return st


def mdot_comm_destroy(comm):
    _check(lib().mdot_comm_destroy(comm), "mdot_comm_destroy")


def mdot_solve_sharded_2d(row_comm, col_comm, row0, n_rows, col0, n_cols, C_block=None, r=None, c=None, *, n,
                          X_block=None, Y_block=None, scale=0.0, recipe="diff",
                          schedule=None, options=None, u_local_out=None, v_local_out=None, check=True):
    """2-D (row x column) sharded solve (include/mdot.h mdot_solve_sharded_2d):
    C_block = C[row0:row0+n_rows, col0:col0+n_cols] (contiguous fp32), or the
    on-the-fly cost's X_block = X[row0:row0+n_rows], Y_block = Y[col0:col0+n_cols];
    r, c the full marginals, n the global size; row_comm joins the ranks of
    this row block, col_comm those of this column block."""
    if C_block is not None:
        if tuple(C_block.shape) != (int(n_rows), int(n_cols)):
            raise ValueError(f"C_block shape {tuple(C_block.shape)} != ({n_rows}, {n_cols})")
    elif X_block is None or Y_block is None or X_block.shape[0] != int(n_rows) or Y_block.shape[0] != int(n_cols):
        raise ValueError("on-the-fly cost: X_block [n_rows x d] and Y_block [n_cols x d] required")
    pb = problem(C_block, r, c, X=X_block, Y=Y_block, scale=scale, n=n, recipe=recipe)
    sched = schedule if schedule is not None else globals()["schedule"]()
    opts = options if options is not None else globals()["options"]()
    if pb.mem == MDOT_MEM_DEVICE:
        opts.stream = _current_stream()
    res = Result()
    dev = pb.mem == MDOT_MEM_DEVICE
    st = lib().mdot_solve_sharded_2d(row_comm, col_comm, ct.byref(pb), int(row0), int(n_rows), int(col0),
                                     int(n_cols), ct.byref(sched), ct.byref(opts),
                                     _ptr(u_local_out, F64, "u_local_out", dev),
                                     _ptr(v_local_out, F64, "v_local_out", dev), ct.byref(res))
    d = res.as_dict()
    d["status"] = st
    if check:
        _check(st, "mdot_solve_sharded_2d")
    return d


def mdot_solve_sharded(comm, row0, n_local, C_local=None, r=None, c=None, *, X_local=None, Y=None,
                       scale=0.0, n=None, schedule=None, options=None, u_local_out=None, v_out=None,
                       check=True, recipe="diff"):
    pb = problem(C_local, r, c, X=X_local, Y=Y, scale=scale, n=n if n is not None else len(c), recipe=recipe)
    sched = schedule if schedule is not None else globals()["schedule"]()
    opts = options if options is not None else globals()["options"]()
    if pb.mem == MDOT_MEM_DEVICE:
        opts.stream = _current_stream()
    res = Result()
    dev = pb.mem == MDOT_MEM_DEVICE
    st = lib().mdot_solve_sharded(comm, ct.byref(pb), int(row0), int(n_local), ct.byref(sched),
                                  ct.byref(opts), _ptr(u_local_out, F64, "u_local_out", dev),
                                  _ptr(v_out, F64, "v_out", dev), ct.byref(res))
    d = res.as_dict()
    d["status"] = st
    if check:
        _check(st, "mdot_solve_sharded")
    return d
