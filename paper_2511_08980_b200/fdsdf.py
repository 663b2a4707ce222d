"""Thin ctypes binding of libfdsdf.so (include/fdsdf.h).

Argument marshalling only: every step of the FD curvature path runs in the CUDA kernels of
csrc/.  torch is used for device memory and streams.  There is no CPU fallback: a missing
library or a non-sm_100 device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# FDSDF_LIB: an alternative build of the same library (A/B timing of compile-time variants)
LIB_PATH = os.environ.get("FDSDF_LIB") or os.path.join(_PKG, "libfdsdf.so")

MAX_LINEAR = 16
ACT = {"softplus": 0, "sine": 1}
FRAME_RANDOM, FRAME_GIVEN = 0, 1
DENOM = {"paper": 0, "one": 1, "grad": 2}
KIND = {"ncr": 0, "nsh": 1}
FD_FORM = {"abs": 0, "square": 1}
STEP_ACCUMULATE, STEP_ALLREDUCE = 1, 2
CREATE_EVAL_ONLY, CREATE_FFMA, CREATE_TENSOR, CREATE_WGRAD_BF16X3 = 1, 2, 4, 8
PATH = {0: "ffma", 1: "tensor", 2: "hybrid"}
FLAG_NONFINITE_INPUT, FLAG_NONFINITE_LOSS, FLAG_ALL_FD_SKIPPED, FLAG_NONFINITE_GRAD = 1, 2, 4, 8
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_EMPTY", 3: "E_CUDA", 4: "E_NCCL", 5: "E_NOMEM",
          6: "E_UNSUPPORTED"}


class FdsdfError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        self.code = STATUS.get(status, str(status))
        super().__init__(f"fdsdf {self.code}: {msg}")


class MlpSpec(C.Structure):
    _fields_ = [("n_linear", C.c_int32), ("width", C.c_int32 * (MAX_LINEAR + 1)), ("act", C.c_int32),
                ("beta", C.c_float), ("omega0_first", C.c_float), ("omega0_hidden", C.c_float),
                ("skip_at", C.c_int32)]


class Stencil(C.Structure):
    _fields_ = [("h", C.c_float), ("frame_seed", C.c_uint64), ("index_offset", C.c_int64),
                ("frame_mode", C.c_int32), ("d_frames_in", C.c_void_p), ("eps_grad", C.c_float),
                ("denom", C.c_int32), ("denom_pow", C.c_int32), ("n_surface", C.c_int64)]


class EvalOut(C.Structure):
    _fields_ = [("d_f", C.c_void_p), ("d_grad", C.c_void_p), ("d_hess", C.c_void_p), ("d_K", C.c_void_p),
                ("d_D", C.c_void_p), ("d_frames", C.c_void_p), ("d_mask", C.c_void_p)]


class Loss(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fd_form", C.c_int32), ("w_dm", C.c_float), ("lambda_dnm", C.c_float),
                ("alpha_dnm", C.c_float), ("lambda_eik", C.c_float), ("lambda_fd", C.c_float),
                ("n_surface_global", C.c_int64), ("n_uniform_global", C.c_int64), ("n_global", C.c_int64)]


_lib = None


def lib():
    """Load libfdsdf.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FdsdfError(6, f"{LIB_PATH} not built (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, u32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
        L.fdsdf_create.argtypes = [C.POINTER(MlpSpec), C.c_int, i64, u32, C.POINTER(vp)]
        L.fdsdf_create.restype = C.c_int
        L.fdsdf_validate_spec.argtypes = [C.POINTER(MlpSpec)]
        L.fdsdf_validate_spec.restype = C.c_int
        L.fdsdf_destroy.argtypes = [vp]
        L.fdsdf_destroy.restype = None
        L.fdsdf_spec_num_params.argtypes = [C.POINTER(MlpSpec)]
        L.fdsdf_spec_num_params.restype = i64
        L.fdsdf_spec_param_offset.argtypes = [C.POINTER(MlpSpec), C.c_int, C.c_int]
        L.fdsdf_spec_param_offset.restype = i64
        L.fdsdf_num_params.argtypes = [vp]
        L.fdsdf_num_params.restype = i64
        L.fdsdf_eval.argtypes = [vp, vp, vp, i64, C.POINTER(Stencil), C.POINTER(EvalOut), vp]
        L.fdsdf_eval.restype = C.c_int
        L.fdsdf_eval_hessian.argtypes = [vp, vp, vp, i64, C.c_float, vp, vp, vp, vp]
        L.fdsdf_eval_hessian.restype = C.c_int
        L.fdsdf_step.argtypes = [vp, vp, vp, i64, C.POINTER(Stencil), C.POINTER(Loss), vp, vp, u32, vp]
        L.fdsdf_step.restype = C.c_int
        L.fdsdf_step_host.argtypes = [vp, vp, vp, i64, C.POINTER(Stencil), C.POINTER(Loss), vp, vp, u32, vp]
        L.fdsdf_step_host.restype = C.c_int
        L.fdsdf_comm_unique_id.argtypes = [C.c_char_p]
        L.fdsdf_comm_unique_id.restype = C.c_int
        L.fdsdf_comm_init.argtypes = [vp, C.c_char_p, C.c_int, C.c_int]
        L.fdsdf_comm_init.restype = C.c_int
        L.fdsdf_allreduce.argtypes = [vp, vp, i64, vp]
        L.fdsdf_allreduce.restype = C.c_int
        L.fdsdf_status_string.argtypes = [C.c_int]
        L.fdsdf_status_string.restype = C.c_char_p
        L.fdsdf_last_error.argtypes = [vp]
        L.fdsdf_last_error.restype = C.c_char_p
        L.fdsdf_get_device_flags.argtypes = [vp, C.POINTER(u32)]
        L.fdsdf_get_device_flags.restype = C.c_int
        L.fdsdf_sample.argtypes = [vp, vp, i64, i64, C.c_float, i64, C.c_uint64, i64, vp, vp]
        L.fdsdf_sample.restype = C.c_int
        L.fdsdf_adam.argtypes = [vp, vp, vp, vp, vp, i64, C.c_float, C.c_float, C.c_float, C.c_float, vp]
        L.fdsdf_adam.restype = C.c_int
        L.fdsdf_path.argtypes = [vp]
        L.fdsdf_path.restype = i32
        L.fdsdf_last_launch_count.argtypes = [vp]
        L.fdsdf_last_launch_count.restype = i32
        L.fdsdf_set_kernel_timing.argtypes = [vp, C.c_int]
        L.fdsdf_set_kernel_timing.restype = C.c_int
        L.fdsdf_kernel_times.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(i64), C.c_int, C.c_int]
        L.fdsdf_kernel_times.restype = C.c_int
        L.fdsdf_selftest_mma.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.fdsdf_selftest_mma.restype = C.c_int
        L.fdsdf_selftest_mma_pair.argtypes = [vp, vp, vp, C.c_int, C.c_int, vp]
        L.fdsdf_selftest_mma_pair.restype = C.c_int
        L.fdsdf_version.argtypes = []
        L.fdsdf_version.restype = C.c_char_p
        L.fdsdf_eval_field.argtypes = [vp, vp, vp, i64, vp, vp, vp]
        L.fdsdf_eval_field.restype = C.c_int
        f32 = C.c_float
        L.fdsdf_grid_points.argtypes = [C.c_int, C.c_int, C.c_int, f32, f32, f32, f32, vp, vp]
        L.fdsdf_grid_points.restype = C.c_int
        L.fdsdf_mesh_work_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        L.fdsdf_mesh_work_bytes.restype = C.c_size_t
        L.fdsdf_mesh_extract.argtypes = [vp, C.c_int, C.c_int, C.c_int, f32, f32, f32, f32, vp, i64,
                                         C.POINTER(i64), vp, C.c_size_t, vp]
        L.fdsdf_mesh_extract.restype = C.c_int
        L.fdsdf_metrics_work_bytes.argtypes = [i64, i64, i64]
        L.fdsdf_metrics_work_bytes.restype = C.c_size_t
        L.fdsdf_mesh_metrics.argtypes = [vp, i64, vp, vp, i64, i64, C.c_uint64, f32, C.POINTER(C.c_double), vp,
                                         C.c_size_t, vp]
        L.fdsdf_mesh_metrics.restype = C.c_int
        _lib = L
    return _lib


def make_spec(spec: dict) -> MlpSpec:
    """C spec from the plain-dict spec used by the harness."""
    w = list(spec["widths"])
    s = MlpSpec()
    s.n_linear = len(w) - 1
    if len(w) > MAX_LINEAR + 1:
        raise FdsdfError(1, "too many layers")
    for i, v in enumerate(w):
        s.width[i] = int(v)
    s.act = ACT[spec["act"]]
    s.beta = float(spec.get("beta", 100.0))
    s.omega0_first = float(spec.get("omega0_first", 30.0))
    s.omega0_hidden = float(spec.get("omega0_hidden", 30.0))
    s.skip_at = int(spec.get("skip_at", -1))
    return s


def _check(status, ctx=None):
    if status != 0:
        msg = lib().fdsdf_last_error(ctx).decode() if ctx else ""
        raise FdsdfError(status, msg)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ----------------------------------------------------------------------------- same-name thin wrappers

def fdsdf_validate_spec(spec: dict) -> int:
    s = make_spec(spec)
    return lib().fdsdf_validate_spec(C.byref(s))


def fdsdf_spec_num_params(spec: dict) -> int:
    s = make_spec(spec)
    return lib().fdsdf_spec_num_params(C.byref(s))


def fdsdf_create(spec: dict, device: int = 0, max_centers: int = 1 << 16, eval_only: bool = False,
                 path: str | None = None, wgrad_bf16x3: bool = False):
    """path: None (library default: "tensor" where supported, else "hybrid"), "ffma" or "tensor";
    wgrad_bf16x3: FDSDF_CREATE_WGRAD_BF16X3 (include/fdsdf.h)."""
    s = make_spec(spec)
    h = C.c_void_p()
    flags = (CREATE_EVAL_ONLY if eval_only else 0) | {None: 0, "ffma": CREATE_FFMA, "tensor": CREATE_TENSOR}[path]
    flags |= CREATE_WGRAD_BF16X3 if wgrad_bf16x3 else 0
    _check(lib().fdsdf_create(C.byref(s), int(device), int(max_centers), flags, C.byref(h)))
    return h


def fdsdf_destroy(ctx):
    lib().fdsdf_destroy(ctx)


def make_stencil(h, n_surface, frame_seed=0, index_offset=0, frames=None, eps_grad=1e-6, denom="paper",
                 denom_pow=4):
    st = Stencil()
    st.h = float(h)
    st.frame_seed = int(frame_seed) & ((1 << 64) - 1)
    st.index_offset = int(index_offset)
    st.frame_mode = FRAME_GIVEN if frames is not None else FRAME_RANDOM
    st.d_frames_in = None if frames is None else frames.data_ptr()
    st.eps_grad = float(eps_grad)
    st.denom = DENOM[denom] if isinstance(denom, str) else int(denom)
    st.denom_pow = int(denom_pow)
    st.n_surface = int(n_surface)
    return st


def make_loss(cfg: dict, counts):
    ls = Loss()
    ls.kind = KIND[cfg["kind"]]
    ls.fd_form = FD_FORM[cfg.get("fd_form", "abs")]
    ls.w_dm = float(cfg["w_dm"])
    ls.lambda_dnm = float(cfg["lambda_dnm"])
    ls.alpha_dnm = float(cfg.get("alpha_dnm", 100.0))
    ls.lambda_eik = float(cfg["lambda_eik"])
    ls.lambda_fd = float(cfg["lambda_fd"])
    ls.n_surface_global, ls.n_uniform_global, ls.n_global = (int(c) for c in counts)
    return ls


def fdsdf_eval_hessian(ctx, params, x, n, h, H, f=None, g=None, stream=None):
    _check(lib().fdsdf_eval_hessian(ctx, _ptr(params), _ptr(x), int(n), float(h), _ptr(H), _ptr(f), _ptr(g),
                                    _stream(stream)), ctx)


def fdsdf_eval_field(ctx, params, x, n, f, g, stream=None):
    _check(lib().fdsdf_eval_field(ctx, _ptr(params), _ptr(x), int(n), _ptr(f), _ptr(g), _stream(stream)), ctx)


def fdsdf_grid_points(nx, ny, nz, origin, spacing, x, stream=None):
    _check(lib().fdsdf_grid_points(int(nx), int(ny), int(nz), *(float(o) for o in origin), float(spacing), _ptr(x),
                                   _stream(stream)))


def fdsdf_mesh_extract(f_grid, origin, spacing, stream=None):
    """Triangles [T, 3, 3] (device fp32) of the zero level set of the grid values f_grid [nz, ny, nx]
    (include/fdsdf.h fdsdf_mesh_extract); the workspace and output are allocated here."""
    import torch
    nz, ny, nx = (int(d) for d in f_grid.shape)
    work = torch.empty(int(lib().fdsdf_mesh_work_bytes(nx, ny, nz)), dtype=torch.uint8, device=f_grid.device)
    nt = C.c_int64(0)
    args = (_ptr(f_grid.contiguous()), nx, ny, nz, *(float(o) for o in origin), float(spacing))
    st = lib().fdsdf_mesh_extract(*args, None, 0, C.byref(nt), _ptr(work), work.numel(), _stream(stream))
    if st not in (0, 1):
        _check(st)
    tris = torch.empty(max(nt.value, 1), 3, 3, dtype=torch.float32, device=f_grid.device)
    _check(lib().fdsdf_mesh_extract(*args, _ptr(tris), tris.shape[0], C.byref(nt), _ptr(work), work.numel(),
                                    _stream(stream)))
    return tris[:nt.value]


def fdsdf_mesh_metrics(tris, gt, gt_normals, nsample=100_000, seed=0, tau=0.005, stream=None):
    """dict(cd, f1, nc, hausdorff, precision, recall) -- unscaled (include/fdsdf.h fdsdf_mesh_metrics)."""
    import torch
    tris = tris.contiguous()
    gt = gt.contiguous()
    gt_normals = gt_normals.contiguous()
    nt, ng = int(tris.shape[0]), int(gt.shape[0])
    work = torch.empty(max(1, int(lib().fdsdf_metrics_work_bytes(nt, int(nsample), ng))), dtype=torch.uint8,
                       device=tris.device)
    out = (C.c_double * 6)()
    _check(lib().fdsdf_mesh_metrics(_ptr(tris), nt, _ptr(gt), _ptr(gt_normals), ng, int(nsample),
                                    C.c_uint64(int(seed) & ((1 << 64) - 1)), float(tau), out, _ptr(work),
                                    work.numel(), _stream(stream)))
    return dict(zip(("cd", "f1", "nc", "hausdorff", "precision", "recall"), list(out)))


def fdsdf_eval(ctx, params, x, n, stencil: Stencil, out: EvalOut, stream=None):
    _check(lib().fdsdf_eval(ctx, _ptr(params), _ptr(x), int(n), C.byref(stencil), C.byref(out),
                            _stream(stream)), ctx)


def fdsdf_step(ctx, params, x, n, stencil: Stencil, loss: Loss, grad, loss_out, flags=0, stream=None):
    _check(lib().fdsdf_step(ctx, _ptr(params), _ptr(x), int(n), C.byref(stencil), C.byref(loss),
                            _ptr(grad), _ptr(loss_out), int(flags), _stream(stream)), ctx)


def fdsdf_step_host(ctx, params, x_host, n, stencil: Stencil, loss: Loss, grad_host, loss_host, flags=0,
                    stream=None):
    """fdsdf_step with HOST buffers (include/fdsdf.h): x_host [n,3] fp32, grad_host [P] fp32 and
    loss_host [8] fp64 are CPU tensors (pinned for asynchronous copies); params is a CUDA tensor.
    Synchronise the stream before reading grad_host / loss_host."""
    for t in (x_host, grad_host, loss_host):
        if getattr(t, "is_cuda", False):
            raise ValueError("fdsdf_step_host takes host (CPU) buffers for x, grad and loss")
    _check(lib().fdsdf_step_host(ctx, _ptr(params), _ptr(x_host), int(n), C.byref(stencil), C.byref(loss),
                                 _ptr(grad_host), _ptr(loss_host), int(flags), _stream(stream)), ctx)


def fdsdf_sample(ctx, pool, n_pick, box_half, n_uniform, seed, iteration, out, stream=None):
    _check(lib().fdsdf_sample(ctx, _ptr(pool), int(pool.shape[0]) if pool is not None else 0, int(n_pick),
                              float(box_half), int(n_uniform), int(seed) & ((1 << 64) - 1), int(iteration),
                              _ptr(out), _stream(stream)), ctx)


def fdsdf_adam(ctx, params, grad, m, v, t, lr=5e-5, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
    _check(lib().fdsdf_adam(ctx, _ptr(params), _ptr(grad), _ptr(m), _ptr(v), int(t), float(lr), float(beta1),
                            float(beta2), float(eps), _stream(stream)), ctx)


def fdsdf_comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().fdsdf_comm_unique_id(buf))
    return buf.raw


def fdsdf_comm_init(ctx, uid: bytes, rank: int, world: int):
    _check(lib().fdsdf_comm_init(ctx, uid, int(rank), int(world)), ctx)


def fdsdf_allreduce(ctx, buf, count=None, stream=None):
    _check(lib().fdsdf_allreduce(ctx, _ptr(buf), int(buf.numel() if count is None else count),
                                 _stream(stream)), ctx)


def fdsdf_get_device_flags(ctx) -> int:
    v = C.c_uint32()
    _check(lib().fdsdf_get_device_flags(ctx, C.byref(v)), ctx)
    return int(v.value)


def fdsdf_last_launch_count(ctx) -> int:
    return int(lib().fdsdf_last_launch_count(ctx))

KSLOTS = ("pack", "fwd", "bwd", "wgrad", "finalize", "allreduce", "pack_tc", "fwd_centre", "sample", "adam",
          "hess")


def fdsdf_set_kernel_timing(ctx, enable: bool):
    _check(lib().fdsdf_set_kernel_timing(ctx, 1 if enable else 0), ctx)


def fdsdf_kernel_times(ctx, reset: bool = False) -> dict:
    """{slot name: (total ms, launches)} of the event-timed launches since the last reset."""
    n = len(KSLOTS)
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    _check(lib().fdsdf_kernel_times(ctx, ms, cnt, n, 1 if reset else 0), ctx)
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KSLOTS)}

# ----------------------------------------------------------------------------- convenience object


class FDSDF:
    """A context bound to one device: eval() / step() on torch CUDA tensors."""

    def __init__(self, spec: dict, device: int = 0, max_centers: int = 1 << 16, eval_only: bool = False,
                 path: str | None = None, wgrad_bf16x3: bool = False):
        import torch
        self.spec = spec
        self.device = torch.device("cuda", device)
        self.ctx = fdsdf_create(spec, device, max_centers, eval_only, path, wgrad_bf16x3)
        self.path = PATH[int(lib().fdsdf_path(self.ctx))]
        self.P = int(lib().fdsdf_num_params(self.ctx))
        self.max_centers = int(max_centers)

    def close(self):
        if self.ctx is not None:
            fdsdf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _dev(self, a, dtype):
        import torch
        if isinstance(a, np.ndarray):
            a = torch.from_numpy(np.ascontiguousarray(a))
        return a.to(device=self.device, dtype=dtype).contiguous()

    def eval(self, params, x, n_surface, h, frame_seed=0, index_offset=0, frames=None, eps_grad=1e-6,
             denom="paper", denom_pow=4, stream=None, outputs=None):
        """Returns a dict of device tensors: f, g, hess (f_uu, f_uv, f_vv), K, D, frames, mask."""
        import torch
        params = self._dev(params, torch.float32)
        x = self._dev(x, torch.float32).reshape(-1, 3)
        n = x.shape[0]
        fr = None if frames is None else self._dev(frames, torch.float32).reshape(n, 6)
        st = make_stencil(h, n_surface, frame_seed, index_offset, fr, eps_grad, denom, denom_pow)
        dev = self.device
        o = outputs or dict(
            f=torch.empty(n, device=dev), g=torch.empty(n, 3, device=dev), hess=torch.empty(n, 3, device=dev),
            K=torch.empty(n, device=dev), D=torch.empty(n, device=dev), frames=torch.empty(n, 6, device=dev),
            mask=torch.empty(n, dtype=torch.uint8, device=dev))
        out = EvalOut(*(_ptr(o.get(k)) for k in ("f", "g", "hess", "K", "D", "frames", "mask")))
        fdsdf_eval(self.ctx, params, x, n, st, out, stream)
        return o

    def eval_hessian(self, params, x, h, H=None, f=None, g=None, stream=None):
        """World-axis 3x3 FD Hessian (19-point stencil): returns H [n,6] = (xx, xy, xz, yy, yz, zz)
        as a device tensor; optional f [n] / g [n,3] output tensors are filled too."""
        import torch
        params = self._dev(params, torch.float32)
        x = self._dev(x, torch.float32).reshape(-1, 3)
        n = x.shape[0]
        if H is None:
            H = torch.empty(n, 6, device=self.device, dtype=torch.float32)
        fdsdf_eval_hessian(self.ctx, params, x, n, h, H, f, g, stream)
        return H

    def eval_field(self, params, x, f=None, g=None, stream=None):
        """f [n] and grad f [n, 3] (device tensors) at points x (no stencil): fdsdf_eval_field, in
        chunks of max_centers."""
        import torch
        params = self._dev(params, torch.float32)
        x = self._dev(x, torch.float32).reshape(-1, 3)
        n = x.shape[0]
        if f is None:
            f = torch.empty(n, device=self.device, dtype=torch.float32)
        if g is None:
            g = torch.empty(n, 3, device=self.device, dtype=torch.float32)
        for a in range(0, n, self.max_centers):
            b = min(n, a + self.max_centers)
            fdsdf_eval_field(self.ctx, params, x[a:b], b - a, f[a:b], g[a:b], stream)
        return f, g

    def extract_mesh(self, params, res, lo=-1.0, hi=1.0, stream=None):
        """The zero level set of f on a res^3 grid over [lo, hi]^3: (triangles [T,3,3], grid f)."""
        import torch
        sp = (hi - lo) / (res - 1)
        x = torch.empty(res ** 3, 3, device=self.device, dtype=torch.float32)
        fdsdf_grid_points(res, res, res, (lo, lo, lo), sp, x, stream)
        f, _ = self.eval_field(params, x, stream=stream)
        fg = f.reshape(res, res, res)
        return fdsdf_mesh_extract(fg, (lo, lo, lo), sp, stream), fg

    def step(self, params, x, n_surface, h, loss_cfg, counts=None, frame_seed=0, index_offset=0, frames=None,
             eps_grad=None, grad=None, loss=None, accumulate=False, allreduce=False, stream=None):
        """Returns (grad [P] fp32, loss [8] fp64) device tensors.  eps_grad (the degenerate-mask
        threshold) defaults to loss_cfg["eps_grad"] when present, else 1e-6."""
        import torch
        if eps_grad is None:
            eps_grad = loss_cfg.get("eps_grad", 1e-6)
        params = self._dev(params, torch.float32)
        x = self._dev(x, torch.float32).reshape(-1, 3)
        n = x.shape[0]
        if counts is None:
            counts = (n_surface, n - n_surface, n)
        fr = None if frames is None else self._dev(frames, torch.float32).reshape(n, 6)
        st = make_stencil(h, n_surface, frame_seed, index_offset, fr, eps_grad, loss_cfg.get("denom", "paper"),
                          loss_cfg.get("denom_pow", 4))
        ls = make_loss(loss_cfg, counts)
        if grad is None:
            grad = torch.zeros(self.P, device=self.device, dtype=torch.float32)
        if loss is None:
            loss = torch.zeros(8, device=self.device, dtype=torch.float64)
        flags = (STEP_ACCUMULATE if accumulate else 0) | (STEP_ALLREDUCE if allreduce else 0)
        fdsdf_step(self.ctx, params, x, n, st, ls, grad, loss, flags, stream)
        return grad, loss

    def sample(self, pool, n_pick, box_half, n_uniform, seed, iteration, out=None, stream=None):
        """Per-iteration batch on the device: n_pick distinct pool rows + n_uniform box points."""
        import torch
        pool = self._dev(pool, torch.float32).reshape(-1, 3)
        if out is None:
            out = torch.empty(int(n_pick) + int(n_uniform), 3, device=self.device, dtype=torch.float32)
        fdsdf_sample(self.ctx, pool, n_pick, box_half, n_uniform, seed, iteration, out, stream)
        return out

    def adam(self, params, grad, m, v, t, lr=5e-5, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
        """In-place Adam update of the device tensor params (m, v: device moment buffers)."""
        fdsdf_adam(self.ctx, params, grad, m, v, t, lr, beta1, beta2, eps, stream)

    def comm_init(self, uid: bytes, rank: int, world: int):
        fdsdf_comm_init(self.ctx, uid, rank, world)

    def device_flags(self) -> int:
        return fdsdf_get_device_flags(self.ctx)

    def launch_count(self) -> int:
        return fdsdf_last_launch_count(self.ctx)

    def set_kernel_timing(self, enable: bool):
        fdsdf_set_kernel_timing(self.ctx, enable)

    def kernel_times(self, reset: bool = False) -> dict:
        return fdsdf_kernel_times(self.ctx, reset)


def fdsdf_selftest_mma(W, B, nprod=6, mn_major=0, stream=None):
    """D = W @ B.T on the tcgen05 bf16-piece core (W [M,K], B [N,K] fp32 CUDA tensors)."""
    import torch
    M, K = W.shape
    N = B.shape[0]
    D = torch.empty(M, N, device=W.device, dtype=torch.float32)
    _check(lib().fdsdf_selftest_mma(_ptr(W.contiguous()), _ptr(B.contiguous()), _ptr(D), M, N, K, int(nprod),
                                    int(mn_major), _stream(stream)))
    return D


def fdsdf_selftest_mma_pair(W, B, stream=None):
    """D = W @ B.T on a tcgen05 CTA pair (W [256,K], B [N,K] fp32 CUDA tensors)."""
    import torch
    N, K = B.shape
    D = torch.empty(256, N, device=W.device, dtype=torch.float32)
    _check(lib().fdsdf_selftest_mma_pair(_ptr(W.contiguous()), _ptr(B.contiguous()), _ptr(D), N, K,
                                         _stream(stream)))
    return D


def version() -> str:
    return lib().fdsdf_version().decode()


class Trainer:
    """The full training iteration of PAPER.md §4 on one device: per
    iteration fdsdf_sample (n_pick of the surface pool + n_uniform box points) ->
    fdsdf_step (+ NCCL allreduce when data-parallel) -> fdsdf_adam, all enqueued on one
    stream with no host synchronisation.  Host-side orchestration only."""

    def __init__(self, model: FDSDF, params, pool, n_pick, n_uniform, box_half, h, loss_cfg, seed=0,
                 lr=5e-5, betas=(0.9, 0.999), eps=1e-8, counts=None, index_offset=0, allreduce=False):
        import torch
        self.m = model
        self.params = model._dev(params, torch.float32).clone()
        self.pool = model._dev(pool, torch.float32).reshape(-1, 3)
        self.n_pick, self.n_uniform, self.box_half, self.h = int(n_pick), int(n_uniform), float(box_half), float(h)
        self.loss_cfg, self.seed, self.lr, self.betas, self.eps = loss_cfg, int(seed), lr, betas, eps
        n = self.n_pick + self.n_uniform
        if allreduce and counts is None:
            # the summed loss / gradient of a data-parallel step is the global mean only with the
            # global counts; each rank also needs its own `seed` (the sampler draws the box points
            # from (seed, iteration, row) alone) and index_offset (frames from the global index)
            raise ValueError("Trainer(allreduce=True) needs the global counts (N_s, N_u, N)")
        self.counts = counts if counts is not None else (self.n_pick, self.n_uniform, n)
        self.index_offset, self.allreduce = int(index_offset), bool(allreduce)
        self.x = torch.empty(n, 3, device=model.device, dtype=torch.float32)
        self.grad = torch.zeros(model.P, device=model.device, dtype=torch.float32)
        self.loss = torch.zeros(8, device=model.device, dtype=torch.float64)
        self.mom1 = torch.zeros_like(self.grad)
        self.mom2 = torch.zeros_like(self.grad)
        self.t = 0

    def state_dict(self):
        """Checkpoint of the training state (SURVEY §5 checkpoint / resume): parameters, the
        Adam moments and the iteration counter (which also keys the batch sampler and the
        frame seeds, so a resumed run continues the same sample / frame sequence).  Host
        copies; the caller persists them (e.g. torch.save)."""
        return {"params": self.params.cpu(), "mom1": self.mom1.cpu(), "mom2": self.mom2.cpu(), "t": int(self.t),
                "seed": int(self.seed)}

    def load_state_dict(self, st):
        """Restore a state_dict() checkpoint (shapes must match this model)."""
        for k in ("params", "mom1", "mom2"):
            src = st[k]
            dst = getattr(self, k)
            if tuple(src.shape) != tuple(dst.shape):
                raise ValueError(f"checkpoint {k} has shape {tuple(src.shape)}, model needs {tuple(dst.shape)}")
            dst.copy_(src.to(dst.device, dst.dtype))
        self.t = int(st["t"])
        self.seed = int(st["seed"])

    def frame_seed(self, it):
        """Per-iteration frame seed: frames are redrawn every iteration; the same
        convention as harness.frame_seed (high 32 bits: base seed, low 32 bits: iteration)."""
        return ((self.seed & 0xFFFFFFFF) << 32 | (int(it) & 0xFFFFFFFF)) & ((1 << 64) - 1)

    def iterate(self, stream=None):
        """One iteration; returns the device loss tensor [8] (of the batch before the update)."""
        it = self.t
        self.m.sample(self.pool, self.n_pick, self.box_half, self.n_uniform, self.seed, it, out=self.x,
                      stream=stream)
        self.m.step(self.params, self.x, self.n_pick, self.h, self.loss_cfg, counts=self.counts,
                    frame_seed=self.frame_seed(it), index_offset=self.index_offset, grad=self.grad,
                    loss=self.loss, allreduce=self.allreduce, stream=stream)
        self.t += 1
        self.m.adam(self.params, self.grad, self.mom1, self.mom2, self.t, self.lr, self.betas[0], self.betas[1],
                    self.eps, stream=stream)
        return self.loss
