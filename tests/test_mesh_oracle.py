"""Pins of the evaluation-side oracle (oracle/mesh_oracle.py): marching
tetrahedra against closed forms and invariants, the counter-based sampler, and the metrics
against SPEC's examples and brute force.  PAPER.md L157 names the metrics."""
import math
import os

import numpy as np
import pytest

from oracle.mesh_oracle import (marching_tetrahedra, counter_u01, sample_mesh, mesh_metrics, triangle_areas,
                                sphere_grid)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _edges(tris, dec=9):
    """undirected edge multiset of a triangle soup, vertices keyed by rounded coordinates"""
    key = lambda v: tuple(np.round(v, dec))  # noqa: E731
    cnt = {}
    for t in tris:
        k = [key(v) for v in t]
        for a, b in ((0, 1), (1, 2), (2, 0)):
            e = tuple(sorted((k[a], k[b])))
            cnt[e] = cnt.get(e, 0) + 1
    return cnt


def test_sphere_mesh_area_position_watertight_and_oriented():
    """|x| - r, r = 0.5 on a 48^3 grid over [-1, 1]^3: total area within 2% of 4 pi r^2,
    every vertex on the sphere to the linear-interpolation error (<< one cell), every edge shared
    by exactly two triangles (the Kuhn split triangulates shared faces identically: watertight),
    every normal pointing outwards (towards f > 0)."""
    f, o, sp = sphere_grid(48)
    tris = marching_tetrahedra(f, o, sp)
    area = triangle_areas(tris).sum()
    assert abs(area - 4 * math.pi * 0.25) < 0.02 * 4 * math.pi * 0.25
    rad = np.linalg.norm(tris.reshape(-1, 3), axis=1)
    assert np.abs(rad - 0.5).max() < 0.25 * sp
    cnt = _edges(tris)
    assert set(cnt.values()) == {2}
    nrm = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0])
    assert np.all((nrm * tris.mean(1)).sum(1) > 0)


def test_plane_mesh_vertices_exact():
    """f = n.x - d is linear: every interpolated vertex lies on the plane to rounding."""
    n = np.array([0.48, -0.6, 0.64])
    sp = 2.0 / 23
    ax = -1.0 + sp * np.arange(24)
    z, y, x = np.meshgrid(ax, ax, ax, indexing="ij")
    f = n[0] * x + n[1] * y + n[2] * z - 0.13
    tris = marching_tetrahedra(f, (-1, -1, -1), sp)
    assert len(tris) > 0
    assert np.abs(tris.reshape(-1, 3) @ n - 0.13).max() < 1e-12
    nrm = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    assert np.abs(nrm @ n - 1.0).max() < 1e-9  # unit normals along +grad f


def test_no_surface_no_triangles_and_single_tet_cases():
    assert len(marching_tetrahedra(np.ones((4, 4, 4)), (0, 0, 0), 1.0)) == 0
    assert len(marching_tetrahedra(-np.ones((4, 4, 4)), (0, 0, 0), 1.0)) == 0
    # one inside corner: the 6 tets of a 2x2x2 grid meeting at corner 0 each cut once
    f = np.ones((2, 2, 2))
    f[0, 0, 0] = -1.0
    tris = marching_tetrahedra(f, (0, 0, 0), 1.0)
    assert len(tris) == 6
    assert np.allclose(np.abs(tris).max(), 0.5)  # every vertex at the edge midpoints t = 1/2


def test_counter_u01_is_the_splitmix64_stream():
    """U(seed, k) = (SplitMix64 output of state seed + (k+1) gamma) >> 11, 2^-53 (golden vector)."""
    want = [int(l) for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and l[0] != "#"]
    u = counter_u01(1234567, [0, 1, 2])
    for a, w in zip(u, want[:3]):
        assert a == (w >> 11) * 2.0 ** -53


def test_sample_mesh_inside_and_area_weighted():
    tri = np.array([[[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[2, 0, 0], [5, 0, 0], [2, 2, 0]]], float)  # areas 0.5, 3
    p, n, t = sample_mesh(tri, 20000, 7)
    assert abs(np.mean(t == 0) - 0.5 / 3.5) < 0.01
    assert np.allclose(np.abs(n[:, 2]), 1.0)
    q = p[t == 0]
    assert q[:, 0].min() >= 0 and q[:, 1].min() >= 0 and (q[:, 0] + q[:, 1]).max() <= 1 + 1e-12
    assert np.allclose(q.mean(0), [1 / 3, 1 / 3, 0], atol=0.01)


def test_metrics_spec_examples():
    """identical sets -> CD 0, F1 1, NC 1, Hausdorff 0; two points at distance d ->
    CD = d = Hausdorff; half of pred within tau and all gt covered -> P = 0.5, R = 1, F1 = 2/3;
    flipped normals -> NC 1 (unoriented); orthogonal normals -> NC 0."""
    rng = np.random.default_rng(1)
    G = rng.uniform(-1, 1, (200, 3))
    Gn = rng.normal(size=(200, 3))
    Gn /= np.linalg.norm(Gn, axis=1, keepdims=True)
    m = mesh_metrics(G, Gn, G, Gn)
    assert m["cd"] == 0 and m["f1"] == 1 and m["nc"] == pytest.approx(1, abs=1e-14) and m["hausdorff"] == 0
    m = mesh_metrics(G, -Gn, G, Gn)
    assert m["nc"] == pytest.approx(1, abs=1e-14)
    e = np.array([[1.0, 0, 0]])
    m = mesh_metrics(np.zeros((1, 3)), e, np.array([[0.3, 0.4, 0.0]]), np.array([[0, 0, 1.0]]))
    assert m["cd"] == pytest.approx(0.5) and m["hausdorff"] == pytest.approx(0.5) and m["nc"] == 0
    P = np.array([[0, 0, 0], [10, 0, 0]], float)
    m = mesh_metrics(P, np.tile(e, (2, 1)), np.zeros((1, 3)), e, tau=0.005)
    assert m["precision"] == 0.5 and m["recall"] == 1.0 and m["f1"] == pytest.approx(2 / 3)


def test_metrics_nearest_neighbours_brute_force():
    """The cKDTree neighbours equal a brute-force O(n^2) search on 500-point sets."""
    rng = np.random.default_rng(2)
    P, G = rng.normal(size=(500, 3)), rng.normal(size=(400, 3))
    Pn = rng.normal(size=(500, 3))
    Pn /= np.linalg.norm(Pn, axis=1, keepdims=True)
    Gn = rng.normal(size=(400, 3))
    Gn /= np.linalg.norm(Gn, axis=1, keepdims=True)
    d = np.linalg.norm(P[:, None] - G[None], axis=2)
    ip, ig = d.argmin(1), d.argmin(0)
    dp, dg = d.min(1), d.min(0)
    cd = 0.5 * (dp.mean() + dg.mean())
    nc = 0.5 * (np.abs((Pn * Gn[ip]).sum(1)).mean() + np.abs((Gn * Pn[ig]).sum(1)).mean())
    m = mesh_metrics(P, Pn, G, Gn, tau=0.3)
    assert m["cd"] == pytest.approx(cd, rel=1e-14) and m["nc"] == pytest.approx(nc, rel=1e-14)
    assert m["hausdorff"] == pytest.approx(max(dp.max(), dg.max()), rel=1e-14)
    assert m["precision"] == np.mean(dp < 0.3) and m["recall"] == np.mean(dg < 0.3)
