"""Pins of the fp64 oracle against what the paper and mathematics fix (not the oracle itself).

Each test names the oracle function it pins and the passage / closed form used.
P:Lx = /root/reference/PAPER.md line x; S:Lx = SPEC.md; App.B = SURVEY.md Appendix B.
"""
import math
import os

import numpy as np
import pytest
import torch

from harness import make_config, mlp_spec, init_params, plane_mlp, num_params
from oracle import (splitmix64, frame_theta, onb, tangent_frames, unflatten, sdf, fd_entries,
                    curvature, loss_terms, oracle_step, oracle_eval, bordered_K,
                    shape_operator_K, hessian_at)

F64 = torch.float64
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _t(a):
    return torch.as_tensor(np.asarray(a, np.float64), dtype=F64)


def _rand_unit(rng, n):
    p = rng.normal(size=(n, 3))
    return p / np.linalg.norm(p, axis=1, keepdims=True)


def _rand_tangent_pair(rng, n):
    """random orthonormal (u, v) not derived from the oracle's ONB."""
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q[:, 0], q[:, 1], np.cross(q[:, 0], q[:, 1])

# ----------------------------------------------------------------------------- frames


def test_splitmix64_reference_vector():
    """pins splitmix64 against the published reference outputs (golden/splitmix64.txt)."""
    want = [int(l) for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and l[0] != "#"]
    x = 1234567
    got = []
    for _ in range(5):
        x = (x + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        got.append(splitmix64(x))
    assert got == want


def test_frame_theta_counter_and_uniformity():
    """theta(seed, i) = 2pi * U where U is the (i+1)-th SplitMix64 output of state=seed;
    uniform on [0, 2pi): circular mean ~ 0."""
    th = frame_theta(1234567, [0, 1, 2])
    want = [int(l) for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and l[0] != "#"]
    for t, w in zip(th, want[:3]):
        assert t == pytest.approx(2 * math.pi * (w >> 11) / 2.0 ** 53, rel=1e-15)
    th = frame_theta(99, range(20000))
    assert th.min() >= 0 and th.max() < 2 * math.pi
    assert abs(np.cos(th).mean()) < 0.02 and abs(np.sin(th).mean()) < 0.02


def test_onb_orthonormal_right_handed():
    """Duff et al. ONB: b1.b2 = b1.n = b2.n = 0, unit norms, det[b1 b2 n] = +1, including
    the poles and the n_z = -0.0 tie (s = +1)."""
    rng = np.random.default_rng(0)
    n = np.concatenate([_rand_unit(rng, 500), [[0, 0, 1], [0, 0, -1], [1, 0, 0],
                                               [0.6, 0.8, -0.0], [0.6, 0.8, 0.0],
                                               [1e-9, 0, -1.0]]])
    n = n / np.linalg.norm(n, axis=1, keepdims=True)
    b1, b2 = onb(_t(n))
    b1, b2, nn = b1.numpy(), b2.numpy(), n
    for a, b in ((b1, b2), (b1, nn), (b2, nn)):
        assert np.abs((a * b).sum(1)).max() < 1e-12
    for a in (b1, b2):
        assert np.abs(np.linalg.norm(a, axis=1) - 1).max() < 1e-12
    det = np.linalg.det(np.stack([b1, b2, nn], 2))
    assert np.abs(det - 1).max() < 1e-12


def test_tangent_frames_invariants_and_mask():
    """(u, v, n) orthonormal and right-handed; masked rows give u = v = 0;
    for a fixed n the frame angle is uniform: mean u ~ 0 over 10k draws."""
    rng = np.random.default_rng(1)
    g = rng.normal(size=(400, 3)) * 3
    mask = torch.ones(400, dtype=torch.bool)
    mask[7] = False
    u, v = tangent_frames(_t(g), mask, 12345, range(400))
    u, v = u.numpy(), v.numpy()
    n = g / np.linalg.norm(g, axis=1, keepdims=True)
    keep = np.arange(400) != 7
    for a, b in ((u, v), (u, n), (v, n)):
        assert np.abs((a * b).sum(1)[keep]).max() < 1e-12
    det = np.linalg.det(np.stack([u, v, n], 2))
    assert np.abs(det[keep] - 1).max() < 1e-12
    assert np.all(u[7] == 0) and np.all(v[7] == 0)
    # fixed normal, many angles
    gg = np.tile([[0.3, -0.5, 0.8]], (10000, 1))
    u, _ = tangent_frames(_t(gg), torch.ones(10000, dtype=torch.bool), 7, range(10000))
    assert np.abs(u.numpy().mean(0)).max() < 0.05
    # axis case (S:L165 example): gradient (0,0,2) -> n = z, u, v in the xy-plane
    u, v = tangent_frames(_t([[0, 0, 2.0]]), torch.ones(1, dtype=torch.bool), 3, [0])
    assert abs(float(u[0, 2])) < 1e-15 and abs(float(v[0, 2])) < 1e-15

# ----------------------------------------------------------------------------- stencils


def test_quadratic_exactness_any_h():
    """f = 1/2 x^T A x + b.x + c: FD gives u^T A u, v^T A v, u^T A v exactly for every h
    (fourth derivatives vanish)."""
    rng = np.random.default_rng(2)
    A = rng.normal(size=(3, 3))
    A = A + A.T
    b = rng.normal(size=3)
    field = lambda x: 0.5 * ((x @ _t(A)) * x).sum(1) + x @ _t(b) + 0.7  # noqa: E731
    x0 = rng.uniform(-1, 1, (50, 3))
    for h in (1e-1, 1e-2, 1e-3):
        u, v, _ = _rand_tangent_pair(rng, 1)
        U = np.tile(u, (50, 1))
        V = np.tile(v, (50, 1))
        fuu, fvv, fuv = fd_entries(field, _t(x0), _t(U), _t(V), h)
        fmax = 10.0
        tol = 64 * 2.2e-16 * fmax / h ** 2
        assert np.abs(fuu.numpy() - u @ A @ u).max() < tol
        assert np.abs(fvv.numpy() - v @ A @ v).max() < tol
        assert np.abs(fuv.numpy() - u @ A @ v).max() < tol


def test_spec_quadratic_example():
    """f = x^T diag(1,2,3) x, u = x, v = y -> (f_uu, f_vv, f_uv) = (2, 4, 0), D = 8."""
    field = lambda x: x[:, 0] ** 2 + 2 * x[:, 1] ** 2 + 3 * x[:, 2] ** 2  # noqa: E731
    fuu, fvv, fuv = fd_entries(field, _t([[0.1, -0.2, 0.3]]), _t([[1, 0, 0]]), _t([[0, 1, 0]]), 0.01)
    assert float(fuu) == pytest.approx(2, abs=1e-9)
    assert float(fvv) == pytest.approx(4, abs=1e-9)
    assert float(fuv) == pytest.approx(0, abs=1e-9)
    D, _ = curvature(fuu, fvv, fuv, _t([1.0]), torch.ones(1, dtype=torch.bool), "one",
                     torch.ones(1, dtype=torch.bool))
    assert float(D) == pytest.approx(8, abs=1e-8)


def test_mixed_stencil_truncation_x3y():
    """f = x^3 y: FD f_xy = 3x^2 + h^2 exactly (App.B corrected constant);
    f_xx = 6xy exactly; f_yy = 0."""
    field = lambda x: x[:, 0] ** 3 * x[:, 1]  # noqa: E731
    x0 = np.array([[0.4, -0.3, 0.2]])
    for h in (1e-1, 3e-2):
        fuu, fvv, fuv = fd_entries(field, _t(x0), _t([[1, 0, 0]]), _t([[0, 1, 0]]), h)
        assert float(fuv) == pytest.approx(3 * 0.4 ** 2 + h * h, abs=1e-12)
        assert float(fuu) == pytest.approx(6 * 0.4 * -0.3, abs=1e-11)
        assert float(fvv) == pytest.approx(0, abs=1e-11)


def test_sphere_exact_fd_and_curvature():
    """Sphere SDF |x| - r: f_uu = f_vv = 2/(sqrt(rho^2+h^2)+rho), f_uv = 0 for any tangent
    frame; r = rho = 0.5, h = 1e-2: D = K = 3.999200199944016 (App.B), and D - 4 ~ -2h^2."""
    r = 0.5
    field = lambda x: torch.linalg.vector_norm(x, dim=1) - r  # noqa: E731
    rng = np.random.default_rng(3)
    x0 = _rand_unit(rng, 64) * r
    X = _t(x0).requires_grad_(True)
    (g,) = torch.autograd.grad(field(X).sum(), X)
    mask = torch.ones(64, dtype=torch.bool)
    u, v = tangent_frames(g, mask, 5, range(64))
    for h, dm4 in ((2e-2, -3.197e-3), (1e-2, -7.998e-4), (5e-3, -2.000e-4), (2.5e-3, -5.000e-5)):
        fuu, fvv, fuv = fd_entries(field, _t(x0), u, v, h)
        want = 2.0 / (math.sqrt(r * r + h * h) + r)
        tol = 1e-15 / h ** 2 * 10
        assert np.abs(fuu.numpy() - want).max() < tol
        assert np.abs(fvv.numpy() - want).max() < tol
        assert np.abs(fuv.numpy()).max() < tol
        gn = torch.linalg.vector_norm(g, dim=1)
        D, K = curvature(fuu, fvv, fuv, gn, mask, "grad", torch.zeros(64, dtype=torch.bool))
        assert np.abs(D.numpy() - 4 - dm4).max() < 2e-3 * abs(dm4) + 20 * tol
        if h == 1e-2:
            assert np.abs(K.numpy() - 3.999200199944016).max() < 1e-9


def test_cylinder_exact_fd():
    """Infinite cylinder sqrt(x^2+y^2) - r at x0 = (0.3, 0.4, 0.1) (App.B): closed forms
    f_uu = 2a_u^2/(S_u+rho), f_vv = 2a_v^2/(S_v+rho), f_uv = 2a_u a_v/(S_+ + S_-);
    printed values (1.169898709750687, 0.829998412231544, -0.985252718270244) at h=1e-2."""
    r, h = 0.5, 1e-2
    field = lambda x: torch.sqrt(x[:, 0] ** 2 + x[:, 1] ** 2) - r  # noqa: E731
    t = np.array([-0.8, 0.6, 0.0])
    z = np.array([0.0, 0.0, 1.0])
    u = math.cos(0.7) * t + math.sin(0.7) * z
    v = -math.sin(0.7) * t + math.cos(0.7) * z
    fuu, fvv, fuv = fd_entries(field, _t([[0.3, 0.4, 0.1]]), _t([u]), _t([v]), h)
    rho = 0.5
    au, av = u @ t, v @ t
    Su, Sv = math.sqrt(rho ** 2 + h * h * au * au), math.sqrt(rho ** 2 + h * h * av * av)
    Sp, Sm = math.sqrt(rho ** 2 + h * h * (au + av) ** 2), math.sqrt(rho ** 2 + h * h * (au - av) ** 2)
    want = (2 * au * au / (Su + rho), 2 * av * av / (Sv + rho), 2 * au * av / (Sp + Sm))
    got = (float(fuu), float(fvv), float(fuv))
    for g_, w_, printed in zip(got, want, (1.169898709750687, 0.829998412231544, -0.985252718270244)):
        assert g_ == pytest.approx(w_, abs=1e-10)
        assert g_ == pytest.approx(printed, abs=1e-10)
    D, _ = curvature(fuu, fvv, fuv, _t([1.0]), torch.ones(1, dtype=torch.bool), "one",
                     torch.ones(1, dtype=torch.bool))
    assert float(D) == pytest.approx(2.912e-4, rel=2e-3)


def test_plane_zero():
    """Plane n.x - d: all FD entries vanish (App.B)."""
    rng = np.random.default_rng(4)
    n = _rand_unit(rng, 1)[0]
    field = lambda x: x @ _t(n) - 0.3  # noqa: E731
    x0 = rng.uniform(-1, 1, (20, 3))
    u, v, _ = _rand_tangent_pair(rng, 1)
    fuu, fvv, fuv = fd_entries(field, _t(x0), _t(np.tile(u, (20, 1))), _t(np.tile(v, (20, 1))), 1e-2)
    for e in (fuu, fvv, fuv):
        assert np.abs(e.numpy()).max() < 1e-11


def test_frame_symmetries():
    """theta -> theta + pi ((u,v) -> (-u,-v)) leaves all three entries unchanged; theta ->
    theta + pi/2 ((u,v) -> (v,-u)) swaps f_uu <-> f_vv, negates f_uv, keeps D (App.B)."""
    spec, params = _tiny_net("sine", 0)
    layers = unflatten(spec, _t(params))
    field = lambda x: sdf(spec, layers, x)  # noqa: E731
    rng = np.random.default_rng(5)
    x0 = _t(rng.uniform(-0.8, 0.8, (16, 3)))
    u, v, _ = _rand_tangent_pair(rng, 1)
    U, V = _t(np.tile(u, (16, 1))), _t(np.tile(v, (16, 1)))
    a = fd_entries(field, x0, U, V, 1e-2)
    b = fd_entries(field, x0, -U, -V, 1e-2)
    c = fd_entries(field, x0, V, -U, 1e-2)
    for p, q in zip(a, b):
        assert torch.allclose(p, q, atol=1e-9, rtol=0)
    assert torch.allclose(a[0], c[1], atol=1e-9) and torch.allclose(a[1], c[0], atol=1e-9)
    assert torch.allclose(a[2], -c[2], atol=1e-9)

# ----------------------------------------------------------------------------- curvature


def test_scaled_sphere_pins_exponent_reading():
    """f = 2(|x| - r), r = 0.5, h = 1e-2 (App.B): D_FD = 15.9968...;
    K_FD with the printed |g|^4 = 0.99980; |g|^2 would give 3.99920; bordered-Hessian K = 4."""
    r, h = 0.5, 1e-2
    field = lambda x: 2 * (torch.linalg.vector_norm(x, dim=1) - r)  # noqa: E731
    x0 = _t([[0.0, 0.3, 0.4]])
    X = x0.clone().requires_grad_(True)
    (g,) = torch.autograd.grad(field(X).sum(), X)
    mask = torch.ones(1, dtype=torch.bool)
    u, v = tangent_frames(g, mask, 1, [0])
    fuu, fvv, fuv = fd_entries(field, x0, u, v, h)
    gn = torch.linalg.vector_norm(g, dim=1)
    D, K = curvature(fuu, fvv, fuv, gn, mask, "grad", torch.zeros(1, dtype=torch.bool))
    fuu_exact = 2 * 2.0 / (math.sqrt(r * r + h * h) + r)
    assert float(D) == pytest.approx(fuu_exact ** 2, abs=1e-8)
    assert float(D) == pytest.approx(15.9968, abs=1e-3)
    assert float(K) == pytest.approx(fuu_exact ** 2 / 16, abs=1e-9)
    assert float(K) == pytest.approx(0.99980, abs=1e-5)
    _, Kp = curvature(fuu, fvv, fuv, gn, mask, "paper", torch.ones(1, dtype=torch.bool))
    assert float(Kp) == pytest.approx(float(D), abs=1e-12)  # near-surface rows: den = 1
    assert bordered_K(field, [0.0, 0.3, 0.4]) == pytest.approx(4.0, abs=1e-9)


def _torus(R, r):
    return lambda x: torch.sqrt((torch.sqrt(x[:, 0] ** 2 + x[:, 1] ** 2) - R) ** 2 + x[:, 2] ** 2) - r


def test_bordered_hessian_closed_forms():
    """bordered_K: sphere r=0.5 -> 4; torus (1, 0.25) outer equator ->
    cos(phi)/(r(R + r cos(phi))) = 3.2; equals det(S_H)/|g|^2 on non-SDF fields
    (App.B) within 1e-9."""
    assert bordered_K(lambda x: torch.linalg.vector_norm(x, dim=1) - 0.5, [0.5, 0, 0]) == \
        pytest.approx(4.0, abs=1e-9)
    assert bordered_K(_torus(1.0, 0.25), [1.25, 0, 0]) == pytest.approx(3.2, abs=1e-9)
    # inner equator: phi = pi -> -1/(0.25*0.75)
    assert bordered_K(_torus(1.0, 0.25), [0.75, 0, 0]) == pytest.approx(-1 / (0.25 * 0.75), abs=1e-9)
    rng = np.random.default_rng(6)
    A = rng.normal(size=(3, 3))
    A = A + A.T
    quad = lambda x: 0.5 * ((x @ _t(A)) * x).sum(1) + x[:, 0] * 0.3  # noqa: E731
    for p in rng.uniform(-1, 1, (5, 3)):
        assert bordered_K(quad, p) == pytest.approx(shape_operator_K(quad, p), abs=1e-9)
        assert bordered_K(_torus(1, 0.3), p) == pytest.approx(shape_operator_K(_torus(1, 0.3), p),
                                                             abs=1e-9)


def test_torus_fd_curvature():
    """FD K on the torus outer equator -> 3.2 within 2%."""
    field = _torus(1.0, 0.25)
    x0 = _t([[1.25 * math.cos(0.4), 1.25 * math.sin(0.4), 0.0]])
    X = x0.clone().requires_grad_(True)
    (g,) = torch.autograd.grad(field(X).sum(), X)
    mask = torch.ones(1, dtype=torch.bool)
    for seed in range(5):
        u, v = tangent_frames(g, mask, seed, [0])
        fuu, fvv, fuv = fd_entries(field, x0, u, v, 1e-2)
        _, K = curvature(fuu, fvv, fuv, torch.linalg.vector_norm(g, dim=1), mask, "grad",
                         torch.zeros(1, dtype=torch.bool))
        assert float(K) == pytest.approx(3.2, rel=0.02)

# ----------------------------------------------------------------------------- MLP


def _tiny_net(act, seed, widths=(3, 8, 8, 1)):
    spec = mlp_spec(list(widths), act, beta=100.0 if act == "softplus" else 1.0)
    return spec, init_params(spec, "siren" if act == "sine" else "xavier", seed).astype(np.float64)


def test_plane_mlp_is_exactly_linear():
    """sp_b(y) - sp_b(-y) = y: the plane MLP computes n.x - d exactly, its gradient is n,
    and all FD entries are 0 (App.B)."""
    n = np.array([0.48, -0.6, 0.64])
    spec, params = plane_mlp(n, 0.1, beta=100.0, hidden_layers=3)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (64, 3)).astype(np.float32)
    o = oracle_eval(spec, params, x, 32, 1e-2, frame_seed=1)
    n32 = n.astype(np.float32).astype(np.float64)
    assert np.abs(o["f"] - (x.astype(np.float64) @ n32 - np.float64(np.float32(0.1)))).max() < 1e-12
    assert np.abs(o["g"] - n32).max() < 1e-12
    for k in ("fuu", "fvv", "fuv", "D", "K"):
        assert np.abs(o[k]).max() < 1e-8


def test_skip_layer_concat_order_and_scale():
    """The skip layer's input is cat(a, x)/sqrt(2) (IGR): with the
    pre-skip layer zeroed and the skip layer reading only the x part scaled by sqrt(2), a
    plane pair reproduces n.x - d exactly; the wrong order or scale would not."""
    n = np.array([0.0, 0.6, 0.8])
    spec = mlp_spec([3, 2, 2, 1], "softplus", beta=100.0, skip_at=1)
    W0 = np.zeros((2, 3)); b0 = np.zeros(2)
    W1 = np.zeros((2, 5)); W1[0, 2:] = math.sqrt(2) * n; W1[1, 2:] = -math.sqrt(2) * n
    b1 = np.zeros(2)
    W2 = np.array([[1.0, -1.0]]); b2 = np.array([-0.2])
    params = np.concatenate([W0.ravel(), b0, W1.ravel(), b1, W2.ravel(), b2])
    assert params.size == num_params(spec)
    x = np.random.default_rng(8).uniform(-1, 1, (32, 3))
    f = sdf(spec, unflatten(spec, _t(params)), _t(x)).numpy()
    assert np.abs(f - (x @ n - 0.2)).max() < 1e-12


def test_softplus_and_sine_special_values():
    """softplus_b(0) = log(2)/b; softplus_b(z) -> z for z >> 1/b; sine layer with W = 0 gives
    sin(omega*b); zero weights everywhere -> f = b_L constant, gradient 0."""
    spec = mlp_spec([3, 1, 1], "softplus", beta=100.0)
    p = np.array([0.0, 0.0, 0.0, 0.0, 1.0, 0.0])  # W0=0,b0=0,W1=1,b1=0
    f = sdf(spec, unflatten(spec, _t(p)), _t([[0.3, 0.2, 0.1]]))
    assert float(f) == pytest.approx(math.log(2) / 100, rel=1e-14)
    p = np.array([0.0, 0.0, 0.0, 5.0, 1.0, 0.0])
    assert float(sdf(spec, unflatten(spec, _t(p)), _t([[0.3, 0.2, 0.1]]))) == pytest.approx(5.0, abs=1e-200)
    spec = mlp_spec([3, 1, 1], "sine", omega0_first=30.0)
    p = np.array([0.0, 0.0, 0.0, 0.05, 2.0, 0.1])
    assert float(sdf(spec, unflatten(spec, _t(p)), _t([[0.3, 0.2, 0.1]]))) == \
        pytest.approx(2 * math.sin(1.5) + 0.1, rel=1e-14)
    spec, params = _tiny_net("sine", 1)
    params[:] = 0
    params[-1] = 0.25
    o = oracle_eval(spec, params.astype(np.float32), np.zeros((4, 3), np.float32), 2, 1e-2)
    assert np.all(o["f"] == 0.25) and np.all(o["g"] == 0) and not o["mask"].any()
    assert np.all(o["fuu"] == 0) and np.all(o["K"] == 0)


@pytest.mark.parametrize("act", ["softplus", "sine"])
def test_gradient_vs_central_differences(act):
    """g = grad_x f agrees with fp64 central differences of f."""
    spec, params = _tiny_net(act, 2)
    x = np.random.default_rng(9).uniform(-0.9, 0.9, (32, 3)).astype(np.float32)
    o = oracle_eval(spec, params.astype(np.float32), x, 16, 1e-2)
    layers = unflatten(spec, _t(params.astype(np.float32)))
    e = 1e-6
    for i in range(3):
        d = np.zeros(3); d[i] = e
        fp = sdf(spec, layers, _t(x.astype(np.float64) + d)).numpy()
        fm = sdf(spec, layers, _t(x.astype(np.float64) - d)).numpy()
        cd = (fp - fm) / (2 * e)
        assert np.abs(cd - o["g"][:, i]).max() < 1e-7 * (1 + np.abs(o["g"]).max())


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_fd_converges_to_mlp_hessian_order_two(name):
    """FD entries -> u^T H u etc. of the analytically differentiated MLP at O(h^2)
    (App. A): err(h)/err(h/2) in [3.5, 4.5]."""
    c = make_config(name, 8, 8)
    spec, params = c["spec"], c["params"].astype(np.float64)
    layers = unflatten(spec, _t(params))
    field = lambda x: sdf(spec, layers, x)  # noqa: E731
    rng = np.random.default_rng(10)
    ratios = []
    for x0 in c["x"][:12].astype(np.float64):
        g, H = hessian_at(field, x0)
        u, v, _ = _rand_tangent_pair(rng, 1)
        exact = np.array([u @ H.numpy() @ u, v @ H.numpy() @ v, u @ H.numpy() @ v])
        errs = []
        for h in (2e-2, 1e-2, 5e-3, 2.5e-3):
            e = fd_entries(field, _t([x0]), _t([u]), _t([v]), h)
            errs.append(np.abs(np.array([float(t) for t in e]) - exact).max())
        ratios += [errs[i] / errs[i + 1] for i in range(3)]
    ratios = np.array(ratios)
    assert 3.5 <= np.median(ratios) <= 4.5
    assert np.mean((ratios >= 3.5) & (ratios <= 4.5)) >= 0.85

# ----------------------------------------------------------------------------- losses


def test_loss_spec_examples():
    """Dirichlet on f = {0.1, -0.1} -> 0.1; eikonal on g = (2,0,0) -> 1 and on
    g = 0 -> 1; DNM with alpha = 100, |f| = 0.05 -> e^-5 = 6.7379e-3."""
    cfg = dict(alpha_dnm=100.0, fd_form="abs", w_dm=1.0, lambda_dnm=1.0, lambda_eik=1.0,
               lambda_fd=1.0)
    f = _t([0.1, -0.1])
    surf = torch.tensor([True, True])
    Z = torch.zeros(2, dtype=F64)
    m = torch.ones(2, dtype=torch.bool)
    dm, dnm, eik, fd, tot = loss_terms(f, _t([1.0, 1.0]), Z, m, surf, cfg, (2, 0, 2))
    assert float(dm) == pytest.approx(0.1, abs=1e-15) and float(eik) == 0 and float(fd) == 0
    _, _, eik, _, _ = loss_terms(_t([0.0]), _t([2.0]), _t([0.0]), m[:1], surf[:1], cfg, (1, 0, 1))
    assert float(eik) == pytest.approx(1.0)
    _, _, eik, _, _ = loss_terms(_t([0.0]), _t([0.0]), _t([0.0]), m[:1], surf[:1], cfg, (1, 0, 1))
    assert float(eik) == pytest.approx(1.0)
    _, dnm, _, _, _ = loss_terms(_t([0.05]), _t([1.0]), _t([0.0]), m[:1], ~surf[:1], cfg, (0, 1, 1))
    assert float(dnm) == pytest.approx(6.7379e-3, rel=1e-4)
    assert float(dnm) == pytest.approx(math.exp(-5), rel=1e-14)


def test_total_loss_linear_in_weights_and_masking():
    """Eq. (1) is linear in (w_dm, lambdas); masked rows contribute 0 to L_fd;
    L_fd uses |Q| (abs) or Q^2 (square)."""
    rng = np.random.default_rng(11)
    f, gn, Q = _t(rng.normal(size=6)), _t(rng.uniform(0.5, 2, 6)), _t(rng.normal(size=6))
    m = torch.tensor([True, True, False, True, True, True])
    s = torch.tensor([True, True, True, False, False, False])
    base = dict(alpha_dnm=100.0, fd_form="abs", w_dm=0.0, lambda_dnm=0.0, lambda_eik=0.0,
                lambda_fd=0.0)
    parts = []
    for k in ("w_dm", "lambda_dnm", "lambda_eik", "lambda_fd"):
        c = dict(base); c[k] = 1.0
        parts.append(float(loss_terms(f, gn, Q, m, s, c, (3, 3, 6))[4]))
    c = dict(base, w_dm=2.0, lambda_dnm=3.0, lambda_eik=5.0, lambda_fd=7.0)
    tot = float(loss_terms(f, gn, Q, m, s, c, (3, 3, 6))[4])
    assert tot == pytest.approx(2 * parts[0] + 3 * parts[1] + 5 * parts[2] + 7 * parts[3], rel=1e-14)
    q = Q.numpy()
    assert parts[3] == pytest.approx(np.abs(q[m.numpy()]).sum() / 6, rel=1e-14)
    c = dict(base, lambda_fd=1.0, fd_form="square")
    assert float(loss_terms(f, gn, Q, m, s, c, (3, 3, 6))[4]) == \
        pytest.approx((q[m.numpy()] ** 2).sum() / 6, rel=1e-14)

# ----------------------------------------------------------------------------- weight gradient (brute force)


LOSS_VARIANTS = [
    dict(kind="ncr", denom="paper", w_dm=1.0, lambda_dnm=100.0, lambda_eik=50.0, lambda_fd=1.0,
         fd_form="abs"),
    dict(kind="ncr", denom="grad", w_dm=0.0, lambda_dnm=0.0, lambda_eik=0.0, lambda_fd=1.0,
         fd_form="abs"),
    dict(kind="nsh", denom="one", w_dm=1.0, lambda_dnm=0.0, lambda_eik=50.0, lambda_fd=1.0,
         fd_form="square"),
]


def _full_cfg(v):
    return dict(v, alpha_dnm=100.0, denom_pow=4, eps_grad=1e-6)


@pytest.mark.parametrize("act", ["softplus", "sine"])
@pytest.mark.parametrize("variant", range(len(LOSS_VARIANTS)))
def test_weight_gradient_brute_force(act, variant):
    """Central FD of the fp64 total loss over EVERY parameter of a tiny net (frames and mask
    frozen) matches oracle_step's gradient: relL2 < 1e-6."""
    spec, params = _tiny_net(act, 3 + variant)
    if act == "softplus":
        spec["beta"] = 10.0
    cfg = _full_cfg(LOSS_VARIANTS[variant])
    x = np.random.default_rng(12 + variant).uniform(-0.8, 0.8, (20, 3)).astype(np.float32)
    p32 = params.astype(np.float32)
    h = float(np.float32(2e-2))  # the oracle promotes the fp32 h exactly
    ref = oracle_step(spec, p32, x, 10, h, cfg, frame_seed=77)
    frames = (ref["u"], ref["v"])
    P = torch.tensor(p32.astype(np.float64), dtype=F64)

    def loss_at(pvec):
        layers = unflatten(spec, pvec)
        X = torch.tensor(x.astype(np.float64), dtype=F64, requires_grad=True)
        field = lambda pts: sdf(spec, layers, pts)  # noqa: E731
        f0 = field(X)
        (g,) = torch.autograd.grad(f0.sum(), X, create_graph=False)
        gn = torch.linalg.vector_norm(g, dim=1)
        m = torch.tensor(ref["mask"])
        fuu, fvv, fuv = fd_entries(field, X.detach(), _t(frames[0]), _t(frames[1]), h)
        s = torch.arange(20) < 10
        D, K = curvature(fuu, fvv, fuv, gn, m, cfg["denom"], s)
        Q = K if cfg["kind"] == "ncr" else D
        return float(loss_terms(f0, gn, Q, m, s, cfg, (10, 10, 20))[4].detach())

    assert loss_at(P) == pytest.approx(ref["loss"][4], rel=1e-12)
    fd = np.empty(P.numel())
    for i in range(P.numel()):
        e = 1e-6 * max(1.0, abs(float(P[i])))
        Pp, Pm = P.clone(), P.clone()
        Pp[i] += e
        Pm[i] -= e
        fd[i] = (loss_at(Pp) - loss_at(Pm)) / (2 * e)
    g = ref["grad"]
    assert np.linalg.norm(fd - g) / np.linalg.norm(g) < 1e-6


def test_output_bias_invariance():
    """f_uu, f_vv, f_uv and g do not depend on b_L, so dL_fd/db_L = dL_eik/db_L = 0 exactly
    (App.B gradient invariants); with lambda_fd = 0 the FD path contributes nothing."""
    spec, params = _tiny_net("sine", 9)
    x = np.random.default_rng(13).uniform(-0.8, 0.8, (16, 3)).astype(np.float32)
    cfg = _full_cfg(dict(kind="ncr", denom="grad", w_dm=0.0, lambda_dnm=0.0, lambda_eik=50.0,
                         lambda_fd=1.0, fd_form="abs"))
    o = oracle_step(spec, params.astype(np.float32), x, 8, 1e-2, cfg, frame_seed=3)
    assert abs(o["grad"][-1]) <= 1e-12 * np.linalg.norm(o["grad"])
    c0 = dict(cfg, lambda_fd=0.0)
    c1 = dict(cfg, lambda_fd=0.0, kind="nsh", fd_form="square")
    a = oracle_step(spec, params.astype(np.float32), x, 8, 1e-2, c0, frame_seed=3)
    b = oracle_step(spec, params.astype(np.float32), x, 8, 1e-2, c1, frame_seed=3)
    assert np.array_equal(a["grad"], b["grad"])
