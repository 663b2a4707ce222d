"""ctypes front end of the plain single-threaded fp64 C oracle (oracle/c/fdsdf_oracle.c).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Argument marshalling only: every step of
the oracle's arithmetic is in the C file (cited there line by line).  The
returned dicts have the same keys as the PyTorch oracle's (oracle/fdsdf_oracle.py), so tests can
run both against the same pins and use either as the GPU parity reference.

`threads` > 1 splits the rows into contiguous chunks, runs the (single-threaded) C function on
each chunk in its own Python thread (ctypes releases the GIL) and adds the chunks' loss sums and
gradients in chunk order: only the test harness parallelises, the oracle itself never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "fdsdf_oracle.c")
LIB = os.path.join(HERE, "c", "libfdsdf_oracle.so")
CFLAGS = ["-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math", "-Wall"]

MAXL = 16
NOUT = 16
ACT = {"softplus": 0, "sine": 1}
FIELD = {"mlp": 0, "sphere": 1, "quadratic": 2, "cylinder": 3, "torus": 4}
KIND = {"ncr": 0, "nsh": 1}
DENOM = {"paper": 0, "one": 1, "grad": 2}
FDFORM = {"abs": 0, "square": 1}


class _Spec(C.Structure):
    _fields_ = [("n_linear", C.c_int), ("width", C.c_int * (MAXL + 1)), ("act", C.c_int),
                ("beta", C.c_double), ("omega_first", C.c_double), ("omega_hidden", C.c_double),
                ("skip_at", C.c_int), ("field", C.c_int), ("fp", C.c_double * 16)]


class _Loss(C.Structure):
    _fields_ = [("kind", C.c_int), ("denom", C.c_int), ("denom_pow", C.c_int), ("fd_form", C.c_int),
                ("eps_grad", C.c_double), ("w_dm", C.c_double), ("lambda_dnm", C.c_double),
                ("alpha_dnm", C.c_double), ("lambda_eik", C.c_double), ("lambda_fd", C.c_double),
                ("n_surface_global", C.c_double), ("n_uniform_global", C.c_double),
                ("n_global", C.c_double)]


def build_lib(force: bool = False) -> str:
    """gcc the oracle into oracle/c/libfdsdf_oracle.so (plain C99, -O2, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.run(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = C.CDLL(build_lib())
        dp = C.POINTER(C.c_double)
        lib.or_step.argtypes = [C.POINTER(_Spec), dp, dp, C.c_int64, C.POINTER(C.c_ubyte), C.c_double,
                                C.POINTER(_Loss), C.c_uint64, C.POINTER(C.c_int64), dp, dp, dp, dp]
        lib.or_step.restype = C.c_int
        lib.or_hessian.argtypes = [C.POINTER(_Spec), dp, dp, C.c_int64, C.c_double, dp, dp]
        lib.or_hessian.restype = C.c_int
        lib.or_num_params.argtypes = [C.POINTER(_Spec)]
        lib.or_num_params.restype = C.c_longlong
        lib.or_frame_theta.argtypes = [C.c_uint64, C.c_int64]
        lib.or_frame_theta.restype = C.c_double
        lib.or_frame.argtypes = [dp, C.c_uint64, C.c_int64, dp, dp]
        lib.or_frame.restype = None
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _spec(spec=None, field="mlp", fparams=()):
    s = _Spec()
    if spec is None:  # analytic field: a dummy 1-layer "net" (no parameters used)
        spec = dict(widths=[3, 1], act="softplus", beta=100.0, omega0_first=30.0, omega0_hidden=30.0,
                    skip_at=-1)
    w = spec["widths"]
    assert len(w) - 1 <= MAXL
    s.n_linear = len(w) - 1
    for i, v in enumerate(w):
        s.width[i] = int(v)
    s.act = ACT[spec["act"]]
    s.beta = float(spec["beta"])
    s.omega_first = float(spec["omega0_first"])
    s.omega_hidden = float(spec["omega0_hidden"])
    s.skip_at = int(spec["skip_at"])
    s.field = FIELD[field]
    for i, v in enumerate(fparams):
        s.fp[i] = float(v)
    return s


def _loss(cfg, counts):
    ls = _Loss()
    ls.kind = KIND[cfg["kind"]]
    ls.denom = DENOM[cfg["denom"]]
    ls.denom_pow = int(cfg["denom_pow"])
    ls.fd_form = FDFORM[cfg["fd_form"]]
    ls.eps_grad = float(cfg["eps_grad"])
    for k in ("w_dm", "lambda_dnm", "alpha_dnm", "lambda_eik", "lambda_fd"):
        setattr(ls, k, float(cfg[k]))
    ls.n_surface_global, ls.n_uniform_global, ls.n_global = (float(c) for c in counts)
    return ls


def num_params_c(spec):
    return int(_L().or_num_params(C.byref(_spec(spec))))


def c_frame(g, frame_seed, gidx):
    """(u, v) of the C oracle's frame (O5) for one gradient g [3]."""
    g = np.ascontiguousarray(np.asarray(g, np.float64).reshape(3))
    u, v = np.zeros(3), np.zeros(3)
    _L().or_frame(_dp(g), C.c_uint64(int(frame_seed) & ((1 << 64) - 1)), int(gidx), _dp(u), _dp(v))
    return u, v


def frame_theta_c(frame_seed, gidx):
    return np.array([_L().or_frame_theta(C.c_uint64(int(frame_seed) & ((1 << 64) - 1)), int(i)) for i in gidx])


def _run(s, P, x, surf, h, ls, frame_seed, gidx, frames, need_grad, npar, threads):
    n = x.shape[0]
    lib = _L()
    out = np.zeros((n, NOUT))
    bounds = np.linspace(0, n, max(1, min(threads, n)) + 1).astype(np.int64) if n else np.array([0, 0])

    def chunk(j):
        a, b = int(bounds[j]), int(bounds[j + 1])
        loss = np.zeros(8)
        G = np.zeros(npar) if need_grad else None
        if b > a:
            fr = frames[a:b] if frames is not None else None
            rc = lib.or_step(C.byref(s), _dp(P), _dp(x[a:b]), b - a,
                             surf[a:b].ctypes.data_as(C.POINTER(C.c_ubyte)), h,
                             C.byref(ls) if ls is not None else None, C.c_uint64(frame_seed),
                             gidx[a:b].ctypes.data_as(C.POINTER(C.c_int64)), _dp(fr), _dp(out[a:b]),
                             _dp(loss), _dp(G))
            assert rc == 0, rc
        return loss, G

    nchunks = len(bounds) - 1
    if nchunks == 1:
        res = [chunk(0)]
    else:
        with ThreadPoolExecutor(nchunks) as ex:
            res = list(ex.map(chunk, range(nchunks)))
    loss = np.zeros(8)
    G = np.zeros(npar) if need_grad else None
    for l_, g_ in res:  # fixed chunk order
        loss += l_
        if need_grad:
            G += g_
    return out, loss, G


def _pack(out, loss, G):
    d = dict(f=out[:, 0], g=out[:, 1:4], fuu=out[:, 4], fuv=out[:, 5], fvv=out[:, 6], D=out[:, 7],
             K=out[:, 8], u=out[:, 9:12], v=out[:, 12:15], mask=out[:, 15] != 0, loss=loss)
    if G is not None:
        d["grad"] = G
    return d


def c_oracle_step(spec, params, x, n_surface, h, cfg, frame_seed=0, index_offset=0, frames=None,
                  counts=None, need_grad=True, surface_mask=None, gidx=None, threads=1, promote=True):
    """Same contract as oracle.oracle_step (fp32 inputs promoted exactly).
    promote=False takes params / x / h as float64 as given (brute-force gradient pins)."""
    f32 = np.float32 if promote else np.float64
    x = np.ascontiguousarray(np.asarray(x, f32).astype(np.float64).reshape(-1, 3))
    N = x.shape[0]
    if surface_mask is None:
        surface_mask = np.arange(N) < n_surface
    surf = np.ascontiguousarray(np.asarray(surface_mask, bool).astype(np.uint8))
    if counts is None:
        ns = int(surf.sum())
        counts = (ns, N - ns, N)
    gidx = np.ascontiguousarray(np.arange(index_offset, index_offset + N, dtype=np.int64) if gidx is None
                                else np.asarray(gidx, np.int64))
    P = np.ascontiguousarray(np.asarray(params, f32).astype(np.float64))
    fr = None
    if frames is not None:
        fr = np.ascontiguousarray(np.concatenate([np.asarray(frames[0], np.float64).reshape(-1, 3),
                                                  np.asarray(frames[1], np.float64).reshape(-1, 3)], 1))
    s = _spec(spec)
    assert P.size == num_params_c(spec), (P.size, num_params_c(spec))
    out, loss, G = _run(s, P, x, surf, float(f32(h)), _loss(cfg, counts), int(frame_seed) & ((1 << 64) - 1),
                        gidx, fr, need_grad, P.size, threads)
    return _pack(out, loss, G)


def c_oracle_eval(spec, params, x, n_surface, h, frame_seed=0, index_offset=0, frames=None, eps_grad=1e-6,
                  denom="paper", denom_pow=4, threads=1):
    cfg = dict(kind="ncr", denom=denom, denom_pow=denom_pow, eps_grad=eps_grad, w_dm=0.0, lambda_dnm=0.0,
               lambda_eik=0.0, lambda_fd=0.0, alpha_dnm=100.0, fd_form="abs")
    return c_oracle_step(spec, params, x, n_surface, h, cfg, frame_seed, index_offset, frames,
                         need_grad=False, threads=threads)


def c_field_eval(field, fparams, x, h, frames=None, frame_seed=0, surface_mask=None, denom="paper",
                 denom_pow=4, eps_grad=1e-6):
    """The stencil / frame / curvature code on an analytic field (pins).
    field in {"sphere" (cx, cy, cz, r, scale), "quadratic" (A row-major 9, b 3, c),
    "cylinder" (r, scale), "torus" (R, r)}; x [N,3] float64 (used as given)."""
    x = np.ascontiguousarray(np.asarray(x, np.float64).reshape(-1, 3))
    N = x.shape[0]
    surf = np.zeros(N, np.uint8) if surface_mask is None else np.asarray(surface_mask, bool).astype(np.uint8)
    cfg = dict(kind="ncr", denom=denom, denom_pow=denom_pow, eps_grad=eps_grad, w_dm=0.0, lambda_dnm=0.0,
               lambda_eik=0.0, lambda_fd=0.0, alpha_dnm=100.0, fd_form="abs")
    fr = None
    if frames is not None:
        fr = np.ascontiguousarray(np.concatenate([np.asarray(frames[0], np.float64).reshape(-1, 3),
                                                  np.asarray(frames[1], np.float64).reshape(-1, 3)], 1))
    out, loss, _ = _run(_spec(None, field, fparams), None, x, np.ascontiguousarray(surf), float(h),
                        _loss(cfg, (1, 1, max(N, 1))), int(frame_seed), np.arange(N, dtype=np.int64), fr,
                        False, 0, 1)
    return _pack(out, loss, None)


def c_oracle_hessian(spec, params, x, h):
    """f and the 19-point world-axis FD Hessian [N,6] (fp32 inputs promoted exactly)."""
    x = np.ascontiguousarray(np.asarray(x, np.float32).astype(np.float64).reshape(-1, 3))
    P = np.ascontiguousarray(np.asarray(params, np.float32).astype(np.float64))
    f = np.zeros(x.shape[0])
    H = np.zeros((x.shape[0], 6))
    rc = _L().or_hessian(C.byref(_spec(spec)), _dp(P), _dp(x), x.shape[0], float(np.float32(h)), _dp(f), _dp(H))
    assert rc == 0
    return f, H
