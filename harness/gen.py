"""Seeded synthetic workloads for the FD-curvature neural-SDF step.

Everything here is input generation: MLP specs, parameter initialisation, point
clouds and loss configurations.  Nothing here evaluates the network, builds
frames or stencils, or computes a loss: that arithmetic lives in `oracle/`
(fp64 CPU) and in the CUDA library (GPU), which share no code.

Stand-ins: the paper trains on ABC CAD meshes (PAPER.md L149-150,
§4 "Datasets": 30k surface samples per mesh, 20k per iteration, plus 20k
uniform off-surface samples in the bounding box).  ABC is not available, so a
seeded CSG union of boxes and capped cylinders with the same counts, normalised
to the same domain, stands in for it.

Flat parameter layout (shared contract, include/fdsdf.h): layer-major; for each
linear layer l: W_l row-major [out][in] then b_l[out].  in_l = widths[l] (+3 if
l == skip_at: the skip layer receives cat(a, x)/sqrt(2)).
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "mlp_spec", "layer_shapes", "num_params", "init_params", "plane_mlp",
    "sphere_surface", "uniform_box", "csg_shape", "csg_surface", "csg_surface_normals", "csg_bbox_diag",
    "add_noise", "csg_cutout_surface", "loss_cfg", "frame_seed", "make_config",
    "CONFIG_NAMES",
]

# ----------------------------------------------------------------------------- specs


def mlp_spec(widths, act, beta=100.0, omega0_first=30.0, omega0_hidden=30.0, skip_at=-1):
    """Plain-dict MLP spec.  act in {"softplus", "sine"}; widths[0]=3, widths[-1]=1."""
    return dict(widths=[int(w) for w in widths], act=str(act), beta=float(beta),
                omega0_first=float(omega0_first), omega0_hidden=float(omega0_hidden),
                skip_at=int(skip_at))


def layer_shapes(spec):
    """[(out, in)] per linear layer, following the flat layout contract."""
    w = spec["widths"]
    out = []
    for l in range(len(w) - 1):
        fan_in = w[l] + (3 if l == spec["skip_at"] else 0)
        out.append((w[l + 1], fan_in))
    return out


def num_params(spec):
    return sum(o * i + o for o, i in layer_shapes(spec))


def init_params(spec, scheme, seed):
    """fp32 flat params.  scheme: "xavier" (W ~ U(±sqrt(6/(fan_in+fan_out))), b = 0) or
    "siren" (first W ~ U(±1/fan_in), others U(±sqrt(6/fan_in)/omega0),
    all b ~ U(±1/sqrt(fan_in)))."""
    rng = np.random.default_rng(seed)
    chunks = []
    for l, (o, i) in enumerate(layer_shapes(spec)):
        if scheme == "xavier":
            lim = math.sqrt(6.0 / (i + o))
            W = rng.uniform(-lim, lim, (o, i))
            b = np.zeros(o)
        elif scheme == "siren":
            if l == 0:
                lim = 1.0 / i
            else:
                lim = math.sqrt(6.0 / i) / spec["omega0_hidden"]
            W = rng.uniform(-lim, lim, (o, i))
            bl = 1.0 / math.sqrt(i)
            b = rng.uniform(-bl, bl, o)
        else:
            raise ValueError(scheme)
        chunks += [W.reshape(-1), b]
    return np.concatenate(chunks).astype(np.float32)


def plane_mlp(normal, offset, beta=100.0, hidden_layers=2):
    """A softplus MLP whose function is exactly the plane n.x - d:
    sp_b(y) - sp_b(-y) = y, carried as a 2-neuron pair through every hidden layer."""
    n = np.asarray(normal, np.float64)
    widths = [3] + [2] * hidden_layers + [1]
    spec = mlp_spec(widths, "softplus", beta=beta)
    chunks = [np.stack([n, -n]).reshape(-1), np.zeros(2)]
    for _ in range(hidden_layers - 1):
        chunks += [np.array([1.0, -1.0, -1.0, 1.0]), np.zeros(2)]
    chunks += [np.array([1.0, -1.0]), np.array([-float(offset)])]
    return spec, np.concatenate(chunks).astype(np.float32)

# ----------------------------------------------------------------------------- points


def sphere_surface(n, radius, seed):
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    return (p * radius).astype(np.float32)


def uniform_box(n, half, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-half, half, (n, 3)).astype(np.float32)


def _rotation(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def csg_shape(seed):
    """3-6 random boxes / capped cylinders: centres U[-0.45,0.45]^3, half-extents and
    radii U[0.1,0.35], uniformly random rotations."""
    rng = np.random.default_rng(seed)
    k = int(rng.integers(3, 7))
    prims = []
    for _ in range(k):
        kind = "box" if rng.uniform() < 0.5 else "cyl"
        c = rng.uniform(-0.45, 0.45, 3)
        R = _rotation(rng)
        if kind == "box":
            prims.append(dict(kind=kind, c=c, R=R, half=rng.uniform(0.1, 0.35, 3)))
        else:
            prims.append(dict(kind=kind, c=c, R=R, r=rng.uniform(0.1, 0.35),
                              hh=rng.uniform(0.1, 0.35)))
    return prims


def _area(p):
    if p["kind"] == "box":
        hx, hy, hz = p["half"]
        return 8.0 * (hx * hy + hy * hz + hx * hz)
    return 2.0 * math.pi * p["r"] * 2.0 * p["hh"] + 2.0 * math.pi * p["r"] ** 2


def _sample_prim(p, m, rng, normals=False):
    """m points uniform (by area) on the surface, local frame (and their outward unit normals)."""
    if p["kind"] == "box":
        h = p["half"]
        face_area = np.array([h[1] * h[2], h[0] * h[2], h[0] * h[1]])
        axis = rng.choice(3, size=m, p=face_area / face_area.sum())
        sgn = np.where(rng.uniform(size=m) < 0.5, -1.0, 1.0)
        loc = rng.uniform(-1.0, 1.0, (m, 3)) * h
        loc[np.arange(m), axis] = sgn * h[axis]
        if normals:
            nrm = np.zeros((m, 3))
            nrm[np.arange(m), axis] = sgn
            return loc, nrm
        return loc
    r, hh = p["r"], p["hh"]
    lat = 2.0 * math.pi * r * 2.0 * hh
    cap = math.pi * r * r
    part = rng.choice(3, size=m, p=np.array([lat, cap, cap]) / (lat + 2 * cap))
    ang = rng.uniform(0, 2 * math.pi, m)
    rad = np.where(part == 0, r, r * np.sqrt(rng.uniform(size=m)))
    z = np.where(part == 0, rng.uniform(-hh, hh, m), np.where(part == 1, hh, -hh))
    loc = np.stack([rad * np.cos(ang), rad * np.sin(ang), z], axis=1)
    if normals:
        nrm = np.stack([np.where(part == 0, np.cos(ang), 0.0), np.where(part == 0, np.sin(ang), 0.0),
                        np.where(part == 0, 0.0, np.where(part == 1, 1.0, -1.0))], axis=1)
        return loc, nrm
    return loc


def _strictly_inside(p, x):
    loc = (x - p["c"]) @ p["R"]
    if p["kind"] == "box":
        return np.all(np.abs(loc) < p["half"], axis=1)
    return (loc[:, 0] ** 2 + loc[:, 1] ** 2 < p["r"] ** 2) & (np.abs(loc[:, 2]) < p["hh"])


def _raw_surface(prims, n, rng, normals=False):
    areas = np.array([_area(p) for p in prims])
    out, outn = [], []
    have = 0
    while have < n:
        m = max(2 * (n - have), 1024)
        which = rng.choice(len(prims), size=m, p=areas / areas.sum())
        pts = np.empty((m, 3))
        nrm = np.empty((m, 3))
        for i, p in enumerate(prims):
            sel = which == i
            if sel.any():
                loc, ln = _sample_prim(p, int(sel.sum()), rng, normals=True)
                pts[sel] = loc @ p["R"].T + p["c"]
                nrm[sel] = ln @ p["R"].T
        keep = np.ones(m, bool)
        for i, p in enumerate(prims):
            keep &= ~(_strictly_inside(p, pts) & (which != i))
        out.append(pts[keep])
        outn.append(nrm[keep])
        have += int(keep.sum())
    if normals:
        return np.concatenate(out)[:n], np.concatenate(outn)[:n]
    return np.concatenate(out)[:n]


def _normaliser(shape_seed):
    prims = csg_shape(shape_seed)
    dense = _raw_surface(prims, 100_000, np.random.default_rng(shape_seed + 1000))
    lo, hi = dense.min(0), dense.max(0)
    centre = 0.5 * (lo + hi)
    scale = 1.8 / float((hi - lo).max())
    return prims, centre, scale, dense


def csg_surface(n, shape_seed, pts_seed):
    """n surface points of the CSG union, normalised so the longest bbox side is 1.8
    (centred at the origin)."""
    prims, centre, scale, _ = _normaliser(shape_seed)
    raw = _raw_surface(prims, n, np.random.default_rng(pts_seed))
    return ((raw - centre) * scale).astype(np.float32)


def csg_surface_normals(n, shape_seed, pts_seed):
    """csg_surface's points (the same draw) and their outward unit normals: the ground truth of the
    reconstruction metrics (normals of the union's primitives, rotated)."""
    prims, centre, scale, _ = _normaliser(shape_seed)
    raw, nrm = _raw_surface(prims, n, np.random.default_rng(pts_seed), normals=True)
    return ((raw - centre) * scale).astype(np.float32), nrm.astype(np.float32)


def csg_bbox_diag(shape_seed):
    _, centre, scale, dense = _normaliser(shape_seed)
    d = (dense - centre) * scale
    return float(np.linalg.norm(d.max(0) - d.min(0)))


def add_noise(points, sigma, seed):
    rng = np.random.default_rng(seed)
    return (points.astype(np.float64) + rng.normal(0.0, sigma, points.shape)).astype(np.float32)


def csg_cutout_surface(n, shape_seed, pts_seed, cut_seed, frac=0.3):
    """Incomplete input (Fig. "incomplete"): drop the 30% of the surface
    beyond a random half-space (threshold = 70th percentile of d.p over a dense sample)."""
    prims, centre, scale, dense = _normaliser(shape_seed)
    rng = np.random.default_rng(cut_seed)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    dn = (dense - centre) * scale
    t = np.percentile(dn @ d, 100.0 * (1.0 - frac))
    out = []
    have = 0
    prng = np.random.default_rng(pts_seed)
    while have < n:
        raw = (_raw_surface(prims, 4 * n, prng) - centre) * scale
        raw = raw[raw @ d <= t]
        out.append(raw)
        have += len(raw)
    return np.concatenate(out)[:n].astype(np.float32)

# ----------------------------------------------------------------------------- losses / frames


def loss_cfg(kind="ncr", denom="paper", w_dm=1.0, lambda_dnm=0.0, lambda_eik=50.0,
             lambda_fd=1.0, alpha_dnm=100.0, fd_form="abs", denom_pow=4, eps_grad=1e-6):
    """Loss configuration (SURVEY §8b fdsdf_loss).  kind: "ncr" (Q = K_FD) or
    "nsh" (Q = D_FD); denom: "paper" (1 on surface rows, |g|^p elsewhere,
    PAPER L131), "one", "grad"."""
    return dict(kind=kind, denom=denom, w_dm=float(w_dm), lambda_dnm=float(lambda_dnm),
                lambda_eik=float(lambda_eik), lambda_fd=float(lambda_fd),
                alpha_dnm=float(alpha_dnm), fd_form=fd_form, denom_pow=int(denom_pow),
                eps_grad=float(eps_grad))


def frame_seed(base, step=0):
    """Per-step frame seed (frames are redrawn every step)."""
    return ((int(base) & 0xFFFFFFFF) << 32 | (int(step) & 0xFFFFFFFF)) & ((1 << 64) - 1)

# ----------------------------------------------------------------------------- configs

CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5")

SIREN_256x4 = dict(widths=[3, 256, 256, 256, 256, 1], act="sine")
SP512x8 = dict(widths=[3, 512, 512, 512, 509, 512, 512, 512, 512, 1], act="softplus", skip_at=4)


def _dflt(v, d):
    return d if v is None else int(v)


def make_config(name, n_surface=None, n_uniform=None, rank=0, h=None):
    """BASELINE.json configs[0..4] (C1..C5) as plain dicts.  n_surface / n_uniform
    override the counts (e.g. the oracle subsample: the first 1024 + 1024 rows)."""
    name = name.lower()
    if name == "c1":
        spec = mlp_spec([3, 64, 64, 1], "softplus", beta=100.0)
        params = init_params(spec, "xavier", 0)
        ns, nu = _dflt(n_surface, 1024), _dflt(n_uniform, 1024)
        xs = sphere_surface(ns, 0.5, 1)
        xu = uniform_box(nu, 1.0, 2)
        loss = loss_cfg("ncr", "paper", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1)
        hh = 1e-2
    elif name in ("c2", "c4", "c5"):
        spec = mlp_spec(**SIREN_256x4)
        params = init_params(spec, "siren", 0)
        if name == "c2":
            ns, nu = _dflt(n_surface, 20_000), _dflt(n_uniform, 20_000)
            # rank r > 0 (data-parallel weak scaling): a fresh draw of the same distribution
            xs = csg_surface(ns, 3, 1 + 1000 * rank)
            xu = uniform_box(nu, 1.1, 2 + 1000 * rank)
            hh = 5e-3
        elif name == "c4":
            ns, nu = _dflt(n_surface, 2_000), _dflt(n_uniform, 20_000)
            xs = csg_cutout_surface(ns, 3, 1, 6)
            xu = uniform_box(nu, 1.1, 2)
            hh = 1e-2
        else:
            ns, nu = _dflt(n_surface, 100_000), _dflt(n_uniform, 100_000)
            xs = csg_surface(ns, 3, 100 + rank)
            xu = uniform_box(nu, 1.1, 200 + rank)
            hh = 5e-3
        loss = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=0, lambda_eik=50, lambda_fd=1)
    elif name == "c3":
        spec = mlp_spec(**SP512x8)
        params = init_params(spec, "xavier", 0)
        ns, nu = _dflt(n_surface, 50_000), _dflt(n_uniform, 50_000)
        xs = csg_surface(ns, 3, 1)
        xs = add_noise(xs, 0.005 * csg_bbox_diag(3), 5)
        xu = uniform_box(nu, 1.1, 2)
        loss = loss_cfg("nsh", "one", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)
        hh = 1e-2
    else:
        raise ValueError(name)
    x = np.concatenate([xs, xu]).astype(np.float32)
    return dict(name=name, spec=spec, params=params, x=x, n_surface=len(xs),
                h=float(np.float32(h if h is not None else hh)), loss=loss,
                frame_seed=frame_seed(4, 0), index_offset=0)
