"""fp64 CPU oracle: the paper's FD curvature losses written out literally.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Plain PyTorch CPU ops in
float64; autograd is used as a library primitive for first derivatives (the
gradient nabla f of PAPER.md L69) and for the weight gradient of the total loss.
No blocking, fusion or reordering: every stencil value is a separate full
evaluation of f at the stencil point formed in fp64, exactly as PAPER.md
L81-91 (§3.1) prints it -- 9 evaluations per centre.

Citation keys: P:Lx = /root/reference/PAPER.md line x; S:Lx = SPEC.md line x;
SURVEY §8c Ox = the oracle step table in SURVEY.md.

Readings of the paper (all listed in DESIGN.md §2):
 * frames: Duff et al. branchless ONB of n = g/|g| (s = +1 when n_z >= 0, incl. -0.0),
   rotated by theta = 2*pi*U with U from SplitMix64(frame_seed, global index)
   ("uniformly random orthogonal completion").  Frames and
   the degenerate mask m = [|g| >= eps] are stop-gradient.
 * masked centres use u = v = 0, so all their FD entries, D and K are exactly 0.
 * K_FD = D_FD / den, den = |g|^p with p = 4 as printed; under the
   "paper" policy den = 1 on surface-role rows.
 * L_DM = mean_surf |f|, L_DNM = mean_unif exp(-alpha|f|), L_eik = mean (|g|-1)^2,
   L_fd = mean m*|Q| (or Q^2), each over the a-priori global counts
   (Eq. 1; forms from S:L278).

Parity unpinned: none of the functions below (see tests/test_oracle_pins.py for
the pin of each).
"""
from __future__ import annotations

import math

import numpy as np
import torch

__all__ = [
    "splitmix64", "frame_theta", "onb", "tangent_frames", "unflatten", "sdf",
    "fd_entries", "curvature", "loss_terms", "oracle_step", "oracle_eval",
    "bordered_K", "shape_operator_K", "hessian_at", "fd_hessian", "oracle_hessian",
]

F64 = torch.float64
_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15

# ----------------------------------------------------------------------------- random frames


def splitmix64(z):
    """SplitMix64 output finaliser (Steele, Lea, Flood 2014) on a python int."""
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def frame_theta(frame_seed, gidx):
    """theta_i = 2*pi * (mix64(seed + (gidx_i + 1)*gamma) >> 11) * 2^-53, fp64
    (SURVEY §8c O5).  gidx: iterable of global centre indices."""
    out = np.empty(len(gidx), np.float64)
    for j, i in enumerate(gidx):
        k = splitmix64((int(frame_seed) + (int(i) + 1) * _GAMMA) & _M64) >> 11
        out[j] = 6.283185307179586 * (float(k) * 2.0 ** -53)
    return out


def onb(n):
    """Branchless right-handed ONB (b1, b2) of unit normals n [M,3] (Duff et al. 2017)."""
    nx, ny, nz = n[:, 0], n[:, 1], n[:, 2]
    s = torch.where(nz >= 0, torch.ones_like(nz), -torch.ones_like(nz))
    a = -1.0 / (s + nz)
    b = nx * ny * a
    b1 = torch.stack([1.0 + s * nx * nx * a, s * b, -s * nx], 1)
    b2 = torch.stack([b, s + ny * ny * a, -ny], 1)
    return b1, b2


def tangent_frames(g, mask, frame_seed, gidx):
    """(u, v) with u x v = n = g/|g| for unmasked centres, (0, 0) for masked ones
    (P:L79).  g is treated as a constant (stop-gradient)."""
    g = g.detach()
    gn = torch.linalg.vector_norm(g, dim=1, keepdim=True)
    n = g / torch.where(gn > 0, gn, torch.ones_like(gn))
    b1, b2 = onb(n)
    th = torch.tensor(frame_theta(frame_seed, gidx), dtype=F64)[:, None]
    u = torch.cos(th) * b1 + torch.sin(th) * b2
    v = -torch.sin(th) * b1 + torch.cos(th) * b2
    m = mask[:, None].to(F64)
    return u * m, v * m

# ----------------------------------------------------------------------------- the SDF MLP


def unflatten(spec, params):
    """Flat params -> [(W [out,in], b [out])] per the layout contract (harness/gen.py)."""
    w = spec["widths"]
    layers, off = [], 0
    for l in range(len(w) - 1):
        fan_in = w[l] + (3 if l == spec["skip_at"] else 0)
        fan_out = w[l + 1]
        W = params[off:off + fan_out * fan_in].reshape(fan_out, fan_in)
        off += fan_out * fan_in
        b = params[off:off + fan_out]
        off += fan_out
        layers.append((W, b))
    assert off == params.numel()
    return layers


def sdf(spec, layers, x):
    """f(x) for points x [M,3].  Hidden layers: SIREN sin(omega*(W a + b)) (omega =
    omega0_first on layer 0, omega0_hidden after) or exact softplus_beta
    (log(1+exp(beta z))/beta, no threshold); last layer linear;
    the skip layer's input is cat(a, x)/sqrt(2) (IGR convention)."""
    a = x
    L = len(layers)
    for l, (W, b) in enumerate(layers):
        if l == spec["skip_at"]:
            a = torch.cat([a, x], dim=1) / math.sqrt(2.0)
        z = a @ W.T + b
        if l == L - 1:
            return z[:, 0]
        if spec["act"] == "sine":
            om = spec["omega0_first"] if l == 0 else spec["omega0_hidden"]
            a = torch.sin(om * z)
        else:
            beta = spec["beta"]
            a = torch.logaddexp(beta * z, torch.zeros_like(z)) / beta
    raise AssertionError

# ----------------------------------------------------------------------------- FD stencils


def fd_entries(field, x0, u, v, h):
    """Central-difference f_uu, f_vv, f_uv at centres x0 [M,3] for a callable field,
    exactly as printed in PAPER.md L83-91: 9 evaluations of f, stencil points formed
    in fp64.  Returns (f_uu, f_vv, f_uv)."""
    f0 = field(x0)
    f_pu = field(x0 + h * u)
    f_mu = field(x0 - h * u)
    f_pv = field(x0 + h * v)
    f_mv = field(x0 - h * v)
    f_pp = field(x0 + h * u + h * v)
    f_pm = field(x0 + h * u - h * v)
    f_mp = field(x0 - h * u + h * v)
    f_mm = field(x0 - h * u - h * v)
    f_uu = (f_pu - 2.0 * f0 + f_mu) / (h * h)
    f_vv = (f_pv - 2.0 * f0 + f_mv) / (h * h)
    f_uv = (f_pp - f_pm - f_mp + f_mm) / (4.0 * h * h)
    return f_uu, f_vv, f_uv


def fd_hessian(field, x0, h):
    """The world-axis 3x3 FD Hessian at centres x0 [M,3] from the 19-point stencil x0,
    x0 +- h e_i, x0 + h(+-e_i +- e_j): the P:L83-91 formulas with
    (u, v) = (e_i, e_j) --
        H_ii = (f(x0 + h e_i) - 2 f(x0) + f(x0 - h e_i)) / h^2
        H_ij = (f(x0 + h e_i + h e_j) - f(x0 + h e_i - h e_j) - f(x0 - h e_i + h e_j)
                + f(x0 - h e_i - h e_j)) / (4 h^2)
    -- every point formed in fp64 and evaluated separately (19 evaluations).
    Returns [M,6] = (H_xx, H_xy, H_xz, H_yy, H_yz, H_zz)."""
    E = torch.eye(3, dtype=x0.dtype)
    f0 = field(x0)
    H = {}
    for i in range(3):
        ei = E[i]
        H[(i, i)] = (field(x0 + h * ei) - 2.0 * f0 + field(x0 - h * ei)) / (h * h)
        for j in range(i + 1, 3):
            ej = E[j]
            H[(i, j)] = (field(x0 + h * ei + h * ej) - field(x0 + h * ei - h * ej)
                         - field(x0 - h * ei + h * ej) + field(x0 - h * ei - h * ej)) / (4.0 * h * h)
    return torch.stack([H[(0, 0)], H[(0, 1)], H[(0, 2)], H[(1, 1)], H[(1, 2)], H[(2, 2)]], dim=1)


def oracle_hessian(spec, params, x, h):
    """f and the 19-point world-axis FD Hessian of the MLP at centres x [N,3] (fp32 inputs
    promoted exactly to fp64).  Returns (f [N], H [N,6]) as numpy fp64."""
    layers = unflatten(spec, torch.as_tensor(np.asarray(params, np.float32), dtype=F64))
    x0 = torch.as_tensor(np.asarray(x, np.float32), dtype=F64).reshape(-1, 3)
    hh = float(np.float32(h))
    field = lambda pts: sdf(spec, layers, pts)  # noqa: E731
    with torch.no_grad():
        return field(x0).numpy(), fd_hessian(field, x0, hh).numpy()


def curvature(f_uu, f_vv, f_uv, gn, mask, den_mode, is_surface, p=4):
    """D_FD = f_uu f_vv - f_uv^2 and K_FD = D_FD/den, den = |g|^p,
    replaced by 1 on near-surface rows under the paper policy.
    Masked rows: K = 0."""
    D = f_uu * f_vv - f_uv * f_uv
    if den_mode == "one":
        den = torch.ones_like(gn)
    else:
        den = gn ** p
        if den_mode == "paper":
            den = torch.where(is_surface, torch.ones_like(den), den)
        elif den_mode != "grad":
            raise ValueError(den_mode)
    den = torch.where(mask, den, torch.ones_like(den))
    K = torch.where(mask, D / den, torch.zeros_like(D))
    return D, K

# ----------------------------------------------------------------------------- Eq. (1)


def loss_terms(f0, gn, Q, mask, is_surface, cfg, counts):
    """(L_DM, L_DNM, L_eik, L_fd, total) with global denominators counts = (N_s, N_u, N)."""
    Ns, Nu, N = counts
    surf = is_surface
    unif = ~is_surface
    zero = f0.sum() * 0.0
    L_dm = (torch.abs(f0[surf]).sum() / Ns) if Ns > 0 else zero
    L_dnm = (torch.exp(-cfg["alpha_dnm"] * torch.abs(f0[unif])).sum() / Nu) if Nu > 0 else zero
    L_eik = ((gn - 1.0) ** 2).sum() / N
    Qm = torch.where(mask, Q, torch.zeros_like(Q))
    if cfg["fd_form"] == "abs":
        L_fd = torch.abs(Qm).sum() / N
    elif cfg["fd_form"] == "square":
        L_fd = (Qm * Qm).sum() / N
    else:
        raise ValueError(cfg["fd_form"])
    total = (cfg["w_dm"] * L_dm + cfg["lambda_dnm"] * L_dnm + cfg["lambda_eik"] * L_eik
             + cfg["lambda_fd"] * L_fd)
    return L_dm, L_dnm, L_eik, L_fd, total

# ----------------------------------------------------------------------------- one step


def oracle_step(spec, params, x, n_surface, h, cfg, frame_seed=0, index_offset=0,
                frames=None, counts=None, need_grad=True, surface_mask=None, gidx=None):
    """One FD-regularised step for centres x [N,3] (fp32 inputs promoted exactly to fp64,
    SURVEY §8c O1).  Rows [0, n_surface) are surface-role.  frames: optional (u, v)
    arrays [N,3] each (GIVEN mode); otherwise random frames from (frame_seed, global
    index = index_offset + row, or the explicit array gidx).  counts: global
    (N_s, N_u, N), default local.  surface_mask: optional bool [N] overriding the
    prefix convention (used by the data-parallel union check).
    Returns a dict of numpy fp64 arrays: f, g, fuu, fuv, fvv, D, K, u, v, mask,
    loss[8] = (dm, dnm, eik, fd, total, n_degenerate, 0, 0) and grad[P] (if need_grad)."""
    x = np.asarray(x, np.float32)
    N = x.shape[0]
    if surface_mask is None:
        surface_mask = np.arange(N) < n_surface
    surface_mask = np.asarray(surface_mask, bool)
    if counts is None:
        ns = int(surface_mask.sum())
        counts = (ns, N - ns, N)
    if gidx is None:
        gidx = range(index_offset, index_offset + N)
    h = float(np.float32(h))
    P = torch.tensor(np.asarray(params, np.float32).astype(np.float64), dtype=F64,
                     requires_grad=need_grad)
    layers = unflatten(spec, P)
    X = torch.tensor(x.astype(np.float64), dtype=F64, requires_grad=True)
    field = lambda pts: sdf(spec, layers, pts)  # noqa: E731

    f0 = field(X)
    (g,) = torch.autograd.grad(f0.sum(), X, create_graph=need_grad)
    gn = torch.linalg.vector_norm(g, dim=1)
    mask = (gn >= cfg["eps_grad"]).detach()
    if frames is None:
        u, v = tangent_frames(g, mask, frame_seed, gidx)
    else:
        u = torch.tensor(np.asarray(frames[0], np.float64), dtype=F64)
        v = torch.tensor(np.asarray(frames[1], np.float64), dtype=F64)
    x0 = X.detach()
    f_uu, f_vv, f_uv = fd_entries(field, x0, u, v, h)
    is_surface = torch.tensor(surface_mask)
    D, K = curvature(f_uu, f_vv, f_uv, gn, mask, cfg["denom"], is_surface, cfg["denom_pow"])
    Q = K if cfg["kind"] == "ncr" else D
    L_dm, L_dnm, L_eik, L_fd, total = loss_terms(f0, gn, Q, mask, is_surface, cfg, counts)
    out = dict(
        f=f0.detach().numpy(), g=g.detach().numpy(),
        fuu=f_uu.detach().numpy(), fuv=f_uv.detach().numpy(), fvv=f_vv.detach().numpy(),
        D=D.detach().numpy(), K=K.detach().numpy(), u=u.numpy(), v=v.numpy(),
        mask=mask.numpy(),
        loss=np.array([float(t.detach()) for t in (L_dm, L_dnm, L_eik, L_fd, total)]
                      + [float((~mask).sum()), 0.0, 0.0]),
    )
    if need_grad:
        (gr,) = torch.autograd.grad(total, P, allow_unused=True)
        out["grad"] = np.zeros(P.numel()) if gr is None else gr.detach().numpy()
    return out


def oracle_eval(spec, params, x, n_surface, h, frame_seed=0, index_offset=0, frames=None,
                eps_grad=1e-6, denom="paper", denom_pow=4):
    """Forward-only quantities (f, g, FD entries, D, K, frames, mask)."""
    cfg = dict(kind="ncr", denom=denom, denom_pow=denom_pow, eps_grad=eps_grad, w_dm=0.0,
               lambda_dnm=0.0, lambda_eik=0.0, lambda_fd=0.0, alpha_dnm=100.0, fd_form="abs")
    return oracle_step(spec, params, x, n_surface, h, cfg, frame_seed, index_offset,
                       frames, need_grad=False)

# ----------------------------------------------------------------------------- analytic references (pins only)


def hessian_at(field, x0):
    """Analytic gradient and Hessian of a scalar field at one point (autograd)."""
    x = torch.as_tensor(x0, dtype=F64).reshape(1, 3).clone().requires_grad_(True)
    f = field(x)
    (g,) = torch.autograd.grad(f.sum(), x, create_graph=True)
    H = torch.stack([torch.autograd.grad(g[0, i], x, retain_graph=True)[0][0] for i in range(3)])
    return g[0].detach(), H.detach()


def bordered_K(field, x0):
    """NRC Gaussian curvature by the bordered Hessian:
    K = -det([[H, g^T], [g, 0]]) / |g|^4."""
    g, H = hessian_at(field, x0)
    B = torch.zeros(4, 4, dtype=F64)
    B[:3, :3] = H
    B[:3, 3] = g
    B[3, :3] = g
    return float(-torch.linalg.det(B) / torch.linalg.vector_norm(g) ** 4)


def shape_operator_K(field, x0):
    """det of the tangent projection of H with an ONB of n, divided by |g|
    -- the shape operator of the level set; equals bordered_K on any field."""
    g, H = hessian_at(field, x0)
    gn = torch.linalg.vector_norm(g)
    b1, b2 = onb((g / gn)[None])
    T = torch.stack([b1[0], b2[0]], 1)
    S = T.T @ H @ T / gn
    return float(torch.linalg.det(S))
