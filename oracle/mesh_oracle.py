"""fp64 CPU oracle of the evaluation side: zero-level-set extraction by
marching tetrahedra and the paper's metrics (§4: "Chamfer Distance (CD, x10^3),
F1 Score (F1, x10^2), and Normal Consistency (NC, x10^2)"), plus the Hausdorff distance of the
Fig. 1 error maps.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  numpy fp64, scipy's cKDTree as the
library nearest-neighbour primitive.

Readings (items 17-21):
 * extraction: marching TETRAHEDRA (each grid cell split into the 6 Kuhn tetrahedra around its
   main diagonal, so neighbouring cells triangulate shared faces identically -- watertight), the
   surface vertex on an edge by linear interpolation t = f_a / (f_a - f_b); inside = f < 0.  The
   paper names no extraction method; SPEC's "marching cubes" is replaced by its table-free
   tetrahedral variant.  Triangles are oriented so their normal points from the inside (f < 0)
   corners to the outside ones.
 * metric samples: `nsample` points area-weighted on the extracted triangles (triangle by inverse
   CDF of the cumulative areas, uniform barycentric point via sqrt), each with the unit face
   normal; the randoms are the counter-based SplitMix64 U(seed, k) of the frame angles.
 * CD = (mean_p d(p, G) + mean_g d(g, P)) / 2 (L2, unsquared); F1 at threshold tau (strict
   d < tau) = 2 P R / (P + R); NC = (mean_p |n_p . n_nn(p)| + mean_g |n_g . n_nn(g)|) / 2
   (unoriented); Hausdorff = max of the two one-sided maxima.  SPEC S:L544-586 (tau = 0.005).

Pins: tests/test_mesh_oracle.py.
"""
from __future__ import annotations

import numpy as np

__all__ = ["KUHN_TETS", "marching_tetrahedra", "counter_u01", "sample_mesh", "mesh_metrics",
           "triangle_areas", "sphere_grid"]

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15

# corner b of a cell = (b & 1, (b >> 1) & 1, (b >> 2) & 1); the 6 Kuhn tetrahedra 0 -> e_i ->
# e_i + e_j -> 7 for the axis orders (i, j, k) below
_ORDERS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
KUHN_TETS = [(0, 1 << i, (1 << i) | (1 << j), 7) for (i, j, k) in _ORDERS]


def _edge(pa, pb, fa, fb):
    t = fa / (fa - fb)
    return pa + t[:, None] * (pb - pa)


def marching_tetrahedra(f, origin, spacing):
    """Triangles [T, 3, 3] (fp64) of the zero level set of grid values f [nz, ny, nx] at points
    origin + spacing * (i, j, k).  Order: cells x-fastest (i + (nx-1)(j + (ny-1) k)), then the 6
    tetrahedra of KUHN_TETS, then up to 2 triangles per tetrahedron."""
    f = np.asarray(f, np.float64)
    nz, ny, nx = f.shape
    o = np.asarray(origin, np.float64)
    kk, jj, ii = np.meshgrid(np.arange(nz - 1), np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    ncell = ii.size
    cf = np.empty((ncell, 8))
    cp = np.empty((ncell, 8, 3))
    for b in range(8):
        dx, dy, dz = b & 1, (b >> 1) & 1, (b >> 2) & 1
        cf[:, b] = f[kk + dz, jj + dy, ii + dx]
        cp[:, b, 0] = o[0] + spacing * (ii + dx)
        cp[:, b, 1] = o[1] + spacing * (jj + dy)
        cp[:, b, 2] = o[2] + spacing * (kk + dz)
    # per cell, per tetrahedron, per slot (0, 1): triangle or nothing
    out = np.full((ncell, 6, 2, 3, 3), np.nan)
    for t, tet in enumerate(KUHN_TETS):
        tf = cf[:, list(tet)]
        tp = cp[:, list(tet)]
        ins = tf < 0.0
        for case in range(16):
            sel = np.all(ins == np.array([(case >> q) & 1 for q in range(4)], bool), axis=1)
            if not sel.any() or case in (0, 15):
                continue
            inside = [q for q in range(4) if (case >> q) & 1]
            outside = [q for q in range(4) if not (case >> q) & 1]
            F, Pp = tf[sel], tp[sel]
            E = lambda a, b: _edge(Pp[:, a], Pp[:, b], F[:, a], F[:, b])  # noqa: E731
            if len(inside) in (1, 3):
                lone = inside[0] if len(inside) == 1 else outside[0]
                oth = [q for q in range(4) if q != lone]
                tris = [(E(lone, oth[0]), E(lone, oth[1]), E(lone, oth[2]))]
            else:
                a, b = inside
                c, d = outside
                tris = [(E(a, c), E(a, d), E(b, d)), (E(a, c), E(b, d), E(b, c))]
            gin = Pp[:, inside].mean(1)
            gout = Pp[:, outside].mean(1)
            for s, (v0, v1, v2) in enumerate(tris):
                nrm = np.cross(v1 - v0, v2 - v0)
                flip = (nrm * (gout - gin)).sum(1) < 0.0
                w1 = np.where(flip[:, None], v2, v1)
                w2 = np.where(flip[:, None], v1, v2)
                out[sel, t, s, 0] = v0
                out[sel, t, s, 1] = w1
                out[sel, t, s, 2] = w2
    out = out.reshape(-1, 3, 3)
    return out[~np.isnan(out[:, 0, 0])]


def splitmix64(z):
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def counter_u01(seed, k):
    """U(seed, k) = (mix64(seed + (k + 1) gamma) >> 11) 2^-53 (the frame angles' generator)."""
    return np.array([float(splitmix64((int(seed) + (int(i) + 1) * _GAMMA) & _M64) >> 11) * 2.0 ** -53
                     for i in np.atleast_1d(k)])


def triangle_areas(tris):
    tris = np.asarray(tris, np.float64)
    return 0.5 * np.linalg.norm(np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0]), axis=1)


def sample_mesh(tris, nsample, seed):
    """nsample points area-weighted on the triangles and their unit face normals: sample s takes
    u0, u1, u2 = U(seed, 3s), U(seed, 3s+1), U(seed, 3s+2); triangle = the first t with
    cumsum(area)[t] > u0 * total; point = (1 - sqrt(u1)) v0 + sqrt(u1)(1 - u2) v1 + sqrt(u1) u2 v2."""
    tris = np.asarray(tris, np.float64)
    area = triangle_areas(tris)
    cum = np.cumsum(area)
    s = np.arange(nsample)
    u = counter_u01(seed, np.stack([3 * s, 3 * s + 1, 3 * s + 2], 1).ravel()).reshape(nsample, 3)
    t = np.searchsorted(cum, u[:, 0] * cum[-1], side="right")
    t = np.minimum(t, len(tris) - 1)
    r1 = np.sqrt(u[:, 1])
    w = np.stack([1.0 - r1, r1 * (1.0 - u[:, 2]), r1 * u[:, 2]], 1)
    tv = tris[t]
    p = (w[:, :, None] * tv).sum(1)
    n = np.cross(tv[:, 1] - tv[:, 0], tv[:, 2] - tv[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    return p, n, t


def mesh_metrics(P, Pn, G, Gn, tau=0.005):
    """CD, F1, NC, Hausdorff (unscaled) and precision / recall between the point samples P (with
    unit normals Pn) and G (Gn) -- nearest neighbours by cKDTree."""
    from scipy.spatial import cKDTree
    P, Pn, G, Gn = (np.asarray(a, np.float64) for a in (P, Pn, G, Gn))
    dp, ip = cKDTree(G).query(P)
    dg, ig = cKDTree(P).query(G)
    prec = float(np.mean(dp < tau))
    rec = float(np.mean(dg < tau))
    f1 = 2.0 * prec * rec / (prec + rec) if prec + rec > 0 else 0.0
    nc = 0.5 * (np.mean(np.abs((Pn * Gn[ip]).sum(1))) + np.mean(np.abs((Gn * Pn[ig]).sum(1))))
    return dict(cd=0.5 * (dp.mean() + dg.mean()), f1=f1, nc=float(nc), hausdorff=float(max(dp.max(), dg.max())),
                precision=prec, recall=rec)


def sphere_grid(res, r=0.5, lo=-1.0, hi=1.0):
    """(f [res]^3 of |x| - r, origin, spacing) -- a pin field"""
    sp = (hi - lo) / (res - 1)
    ax = lo + sp * np.arange(res)
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    return np.sqrt(x * x + y * y + z * z) - r, (lo, lo, lo), sp

