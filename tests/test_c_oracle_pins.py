"""Pins of the plain single-threaded fp64 C oracle (oracle/c/fdsdf_oracle.c) against what the
paper and mathematics fix -- closed forms, invariants, special cases and brute force -- plus the
closed-form pin of the SIREN hidden-layer frequency for BOTH oracles.

P:Lx = /root/reference/PAPER.md line x; S:Lx = SPEC.md; App.B = SURVEY.md Appendix B.
"""
import math
import os

import numpy as np
import pytest

from harness import make_config, mlp_spec, init_params, plane_mlp, num_params, loss_cfg
from oracle import oracle_step, oracle_eval
from oracle.c_oracle import (c_oracle_step, c_oracle_eval, c_field_eval, c_frame, frame_theta_c,
                             num_params_c, c_oracle_hessian)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_unit(rng, n):
    p = rng.normal(size=(n, 3))
    return p / np.linalg.norm(p, axis=1, keepdims=True)


def _rand_tangent_pair(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q[:, 0], q[:, 1]

# ----------------------------------------------------------------------------- frames (O5)


def test_c_frame_theta_golden_and_frame_invariants():
    """theta(seed, i) = 2 pi (mix64(seed + (i+1) gamma) >> 11) 2^-53 against the published
    SplitMix64 outputs (golden/splitmix64.txt: state 1234567); (u, v, n) orthonormal and
    right-handed for random normals and the n_z = +-0 / +-1 edge cases."""
    want = [int(l) for l in open(os.path.join(GOLDEN, "splitmix64.txt")) if l.strip() and l[0] != "#"]
    th = frame_theta_c(1234567, [0, 1, 2])
    for t, w in zip(th, want[:3]):
        assert t == pytest.approx(2 * math.pi * (w >> 11) / 2.0 ** 53, rel=1e-15)
    rng = np.random.default_rng(1)
    gs = list(_rand_unit(rng, 200) * rng.uniform(0.1, 3, (200, 1)))
    gs += [np.array([0, 0, 2.0]), np.array([0, 0, -1.0]), np.array([1.0, 0, 0.0]), np.array([0.3, 0.4, -0.0])]
    for i, g in enumerate(gs):
        u, v = c_frame(g, 99, i)
        n = g / np.linalg.norm(g)
        assert abs(u @ n) < 1e-12 and abs(v @ n) < 1e-12 and abs(u @ v) < 1e-12
        assert abs(np.linalg.norm(u) - 1) < 1e-12 and abs(np.linalg.norm(v) - 1) < 1e-12
        assert np.allclose(np.cross(u, v), n, atol=1e-12)
    th = frame_theta_c(77, range(20000))
    assert abs(np.cos(th).mean()) < 0.02 and abs(np.sin(th).mean()) < 0.02

# ----------------------------------------------------------------------------- stencils on analytic fields


def test_c_quadratic_exactness_and_spec_example():
    """f = 1/2 x^T A x + b.x + c: FD gives u^T A u, v^T A v, u^T A v exactly for every h (S:L217,
    S:L237); S:L217 example diag(2,4,6)/2 with u = x, v = y -> (2, 4, 0), D = 8; A = 0 (a plane)
    -> all entries 0 (App.B)."""
    rng = np.random.default_rng(2)
    A = rng.normal(size=(3, 3))
    A = A + A.T
    b = rng.normal(size=3)
    fp = list(A.ravel()) + list(b) + [0.7]
    x0 = rng.uniform(-1, 1, (50, 3))
    for h in (1e-1, 1e-2, 1e-3):
        u, v = _rand_tangent_pair(rng)
        o = c_field_eval("quadratic", fp, x0, h, frames=(np.tile(u, (50, 1)), np.tile(v, (50, 1))))
        tol = 64 * 2.2e-16 * 10.0 / h ** 2
        assert np.abs(o["fuu"] - u @ A @ u).max() < tol
        assert np.abs(o["fvv"] - v @ A @ v).max() < tol
        assert np.abs(o["fuv"] - u @ A @ v).max() < tol
    fp = [2, 0, 0, 0, 4, 0, 0, 0, 6, 0, 0, 0, 0]
    o = c_field_eval("quadratic", fp, [[0.1, -0.2, 0.3]], 0.01, frames=([[1, 0, 0]], [[0, 1, 0]]),
                     denom="one")
    assert o["fuu"][0] == pytest.approx(2, abs=1e-9) and o["fvv"][0] == pytest.approx(4, abs=1e-9)
    assert o["fuv"][0] == pytest.approx(0, abs=1e-9) and o["D"][0] == pytest.approx(8, abs=1e-8)
    n = _rand_unit(rng, 1)[0]
    o = c_field_eval("quadratic", [0] * 9 + list(n) + [-0.3], rng.uniform(-1, 1, (20, 3)), 1e-2, frame_seed=4)
    for k in ("fuu", "fvv", "fuv", "D", "K"):
        assert np.abs(o[k]).max() < 1e-11
    assert np.abs(o["g"] - n).max() < 1e-15


def test_c_sphere_exact_fd_curvature_and_exponent():
    """Sphere |x| - r (App.B): f_uu = f_vv = 2/(sqrt(rho^2+h^2)+rho), f_uv = 0 for the oracle's own
    random frames; r = 0.5, h = 1e-2: K = 3.999200199944016 and D - 4 ~ -2h^2 -> O(h^2).
    Scaled sphere 2(|x| - r) pins the printed |g|^4 exponent:
    D = 15.9968..., K = D/16 = 0.99980, and 1 on surface rows under the paper policy."""
    r = 0.5
    rng = np.random.default_rng(3)
    x0 = _rand_unit(rng, 64) * r
    for h, dm4 in ((2e-2, -3.197e-3), (1e-2, -7.998e-4), (5e-3, -2.000e-4), (2.5e-3, -5.000e-5)):
        o = c_field_eval("sphere", [0, 0, 0, r, 1.0], x0, h, frame_seed=5, denom="grad")
        want = 2.0 / (math.sqrt(r * r + h * h) + r)
        tol = 1e-14 / h ** 2
        assert np.abs(o["fuu"] - want).max() < tol and np.abs(o["fvv"] - want).max() < tol
        assert np.abs(o["fuv"]).max() < tol
        assert np.abs(o["D"] - 4 - dm4).max() < 2e-3 * abs(dm4) + 20 * tol
        if h == 1e-2:
            assert np.abs(o["K"] - 3.999200199944016).max() < 1e-9
    x = [[0.0, 0.3, 0.4]]
    o = c_field_eval("sphere", [0, 0, 0, r, 2.0], x, 1e-2, frame_seed=1, denom="grad")
    fuu_exact = 2 * 2.0 / (math.sqrt(r * r + 1e-4) + r)
    assert o["D"][0] == pytest.approx(fuu_exact ** 2, abs=1e-8) and o["D"][0] == pytest.approx(15.9968, abs=1e-3)
    assert o["K"][0] == pytest.approx(fuu_exact ** 2 / 16, abs=1e-9) and o["K"][0] == pytest.approx(0.99980, abs=1e-5)
    o = c_field_eval("sphere", [0, 0, 0, r, 2.0], x, 1e-2, frame_seed=1, denom="paper", surface_mask=[True])
    assert o["K"][0] == pytest.approx(o["D"][0], abs=1e-12)


def test_c_cylinder_printed_values_and_torus():
    """Cylinder sqrt(x^2+y^2) - r at (0.3, 0.4, 0.1), h = 1e-2 (App.B closed form, printed
    (1.169898709750687, 0.829998412231544, -0.985252718270244), D_FD = 2.912e-4 = O(h^2));
    torus (R, r) = (1, 0.25) outer equator: FD K -> 3.2 within 2%."""
    t = np.array([-0.8, 0.6, 0.0])
    z = np.array([0.0, 0.0, 1.0])
    u = math.cos(0.7) * t + math.sin(0.7) * z
    v = -math.sin(0.7) * t + math.cos(0.7) * z
    o = c_field_eval("cylinder", [0.5, 1.0], [[0.3, 0.4, 0.1]], 1e-2, frames=([u], [v]), denom="one")
    for k, printed in zip(("fuu", "fvv", "fuv"), (1.169898709750687, 0.829998412231544, -0.985252718270244)):
        assert o[k][0] == pytest.approx(printed, abs=1e-10)
    assert o["D"][0] == pytest.approx(2.912e-4, rel=2e-3)
    x0 = [[1.25 * math.cos(0.4), 1.25 * math.sin(0.4), 0.0]]
    for seed in range(5):
        o = c_field_eval("torus", [1.0, 0.25], x0, 1e-2, frame_seed=seed, denom="grad")
        assert o["K"][0] == pytest.approx(3.2, rel=0.02)

# ----------------------------------------------------------------------------- the MLP


def _sine_closed_form(W, b, om_first, om_hidden, x):
    """f(x) of a sine MLP written out with math.sin, one neuron at a time: layer 0 uses
    om_first, hidden layers om_hidden, last layer linear."""
    a = list(x)
    for l, (Wl, bl) in enumerate(zip(W, b)):
        z = [sum(Wl[i][k] * a[k] for k in range(len(a))) + bl[i] for i in range(len(bl))]
        if l == len(W) - 1:
            return z[0]
        om = om_first if l == 0 else om_hidden
        a = [math.sin(om * zi) for zi in z]


def _sine_closed_grad(W, b, om_first, om_hidden, x):
    """grad f by the chain rule, written out (cos(om z) om W products)."""
    a, J = list(x), np.eye(3)  # J = d a / d x
    for l, (Wl, bl) in enumerate(zip(W, b)):
        Wl = np.array(Wl)
        z = Wl @ np.array(a) + np.array(bl)
        Jz = Wl @ J
        if l == len(W) - 1:
            return Jz[0]
        om = om_first if l == 0 else om_hidden
        a = list(np.sin(om * z))
        J = (om * np.cos(om * z))[:, None] * Jz


@pytest.mark.parametrize("om_first,om_hidden", [(30.0, 15.0), (15.0, 30.0), (30.0, 30.0)])
@pytest.mark.parametrize("impl", ["c", "torch"])
def test_sine_hidden_layer_frequency_closed_form(om_first, om_hidden, impl):
    """Hand-set 3->2->2->1 SIREN with omega0_first != omega0_hidden: f, grad f and the FD entries
    of BOTH oracles equal the closed form written with math.sin (a mix-up of the first / hidden
    frequency, or an omega dropped or applied twice on a hidden layer, fails)."""
    W = [[[0.011, -0.023, 0.017], [0.021, 0.005, -0.013]], [[0.037, -0.029], [-0.019, 0.041]],
         [[0.7, -0.45]]]
    b = [[0.013, -0.007], [0.021, 0.009], [0.05]]
    spec = mlp_spec([3, 2, 2, 1], "sine", omega0_first=om_first, omega0_hidden=om_hidden)
    params = np.concatenate([np.concatenate([np.ravel(Wl), bl]) for Wl, bl in zip(W, b)]).astype(np.float32)
    Wd = [np.array(Wl, np.float32).astype(np.float64).tolist() for Wl in W]
    bd = [np.array(bl, np.float32).astype(np.float64).tolist() for bl in b]
    rng = np.random.default_rng(21)
    x = rng.uniform(-0.9, 0.9, (12, 3)).astype(np.float32)
    u, v = _rand_tangent_pair(rng)
    U, V = np.tile(u, (12, 1)), np.tile(v, (12, 1))
    h = float(np.float32(1e-2))
    ev = (c_oracle_eval if impl == "c" else oracle_eval)(spec, params, x, 6, h, frames=(U, V))
    for i, xi in enumerate(x.astype(np.float64)):
        f = lambda p: _sine_closed_form(Wd, bd, om_first, om_hidden, p)  # noqa: E731
        assert ev["f"][i] == pytest.approx(f(xi), rel=1e-13, abs=1e-15)
        assert np.allclose(ev["g"][i], _sine_closed_grad(Wd, bd, om_first, om_hidden, xi), rtol=1e-12, atol=1e-14)
        fk = [f(xi + h * (cu * u + cv * v)) for cu, cv in ((1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1))]
        f0 = f(xi)
        fuu = (fk[0] - 2 * f0 + fk[1]) / h ** 2
        fvv = (fk[2] - 2 * f0 + fk[3]) / h ** 2
        fuv = (fk[4] - fk[5] - fk[6] + fk[7]) / (4 * h * h)
        tol = 1e-13 * (1 + abs(f0)) / h ** 2
        assert abs(ev["fuu"][i] - fuu) < tol and abs(ev["fvv"][i] - fvv) < tol and abs(ev["fuv"][i] - fuv) < tol


def test_c_plane_mlp_skip_and_zero_weights():
    """Plane MLP (sp(z) - sp(-z) = z) computes n.x - d exactly with gradient n and zero FD
    entries (App.B, T3); the skip layer's input is cat(a, x)/sqrt(2); zero
    weights give the constant b_L with zero gradient."""
    n = np.array([0.48, -0.6, 0.64])
    spec, params = plane_mlp(n, 0.1, beta=100.0, hidden_layers=3)
    x = np.random.default_rng(7).uniform(-1, 1, (64, 3)).astype(np.float32)
    o = c_oracle_eval(spec, params, x, 32, 1e-2, frame_seed=1)
    n32 = n.astype(np.float32).astype(np.float64)
    assert np.abs(o["f"] - (x.astype(np.float64) @ n32 - np.float64(np.float32(0.1)))).max() < 1e-12
    assert np.abs(o["g"] - n32).max() < 1e-12
    for k in ("fuu", "fvv", "fuv", "D", "K"):
        assert np.abs(o[k]).max() < 1e-8
    spec = mlp_spec([3, 2, 2, 1], "softplus", beta=100.0, skip_at=1)
    W0 = np.zeros((2, 3)); b0 = np.zeros(2)
    W1 = np.zeros((2, 5)); W1[0, 2:] = math.sqrt(2) * n; W1[1, 2:] = -math.sqrt(2) * n
    W2 = np.array([[1.0, -1.0]]); b2 = np.array([-0.2])
    p = np.concatenate([W0.ravel(), b0, W1.ravel(), np.zeros(2), W2.ravel(), b2])
    assert p.size == num_params(spec) == num_params_c(spec)
    xx = np.random.default_rng(8).uniform(-1, 1, (32, 3))
    o = c_oracle_step(spec, p, xx, 16, 1e-2, loss_cfg(), promote=False, need_grad=False)
    assert np.abs(o["f"] - (xx @ n - 0.2)).max() < 1e-12
    spec = mlp_spec([3, 8, 8, 1], "sine")
    p = np.zeros(num_params(spec), np.float32)
    p[-1] = 0.25
    o = c_oracle_eval(spec, p, np.zeros((4, 3), np.float32), 2, 1e-2)
    assert np.all(o["f"] == 0.25) and np.all(o["g"] == 0) and not o["mask"].any()
    assert np.all(o["fuu"] == 0) and np.all(o["K"] == 0)


@pytest.mark.parametrize("act", ["softplus", "sine"])
def test_c_gradient_vs_central_differences(act):
    """g = grad_x f agrees with central differences of the oracle's own f."""
    spec = mlp_spec([3, 8, 8, 1], act, beta=100.0, omega0_first=30.0, omega0_hidden=12.0)
    params = init_params(spec, "siren" if act == "sine" else "xavier", 2).astype(np.float64)
    x = np.random.default_rng(9).uniform(-0.9, 0.9, (32, 3))
    cfg = loss_cfg()
    o = c_oracle_step(spec, params, x, 16, 1e-2, cfg, promote=False, need_grad=False)
    e = 1e-6
    for i in range(3):
        d = np.zeros(3); d[i] = e
        fp = c_oracle_step(spec, params, x + d, 16, 1e-2, cfg, promote=False, need_grad=False)["f"]
        fm = c_oracle_step(spec, params, x - d, 16, 1e-2, cfg, promote=False, need_grad=False)["f"]
        assert np.abs((fp - fm) / (2 * e) - o["g"][:, i]).max() < 1e-7 * (1 + np.abs(o["g"]).max())


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_c_fd_converges_to_mlp_hessian_order_two(name):
    """The C oracle's FD entries -> u^T H u etc. of the analytically differentiated MLP (torch
    autograd Hessian, a library primitive) at O(h^2) (App. A):
    err(h)/err(h/2) in [3.5, 4.5]."""
    import torch
    from oracle import unflatten, sdf, hessian_at
    c = make_config(name, 6, 6)
    spec, params = c["spec"], c["params"].astype(np.float64)
    layers = unflatten(spec, torch.tensor(params))
    field = lambda x: sdf(spec, layers, x)  # noqa: E731
    rng = np.random.default_rng(10)
    ratios = []
    for x0 in c["x"][:12].astype(np.float64):
        _, H = hessian_at(field, x0)
        H = H.numpy()
        u, v = _rand_tangent_pair(rng)
        exact = np.array([u @ H @ u, v @ H @ v, u @ H @ v])
        errs = []
        for h in (2e-2, 1e-2, 5e-3, 2.5e-3):
            o = c_oracle_step(spec, params, [x0], 1, h, loss_cfg(), frames=([u], [v]), promote=False,
                              need_grad=False)
            errs.append(np.abs(np.array([o["fuu"][0], o["fvv"][0], o["fuv"][0]]) - exact).max())
        ratios += [errs[i] / errs[i + 1] for i in range(3)]
    ratios = np.array(ratios)
    assert 3.5 <= np.median(ratios) <= 4.5
    assert np.mean((ratios >= 3.5) & (ratios <= 4.5)) >= 0.85

# ----------------------------------------------------------------------------- losses and gradient


def test_c_loss_spec_examples_and_linearity():
    """S:L281-301 on a field with known f and g: Dirichlet on |f| = 0.1 -> 0.1; DNM at
    |f| = 0.05, alpha = 100 -> e^-5; eikonal on |g| = 2 -> 1 (scaled sphere); the total is
    linear in the weights."""
    # sphere s(|x| - r) with s = 2: |g| = 2 everywhere; points at |x| = r +- 0.05 -> f = +-0.1
    x = np.array([[0.55, 0, 0], [0, 0.45, 0]])
    cfg = loss_cfg("ncr", "one", w_dm=1.0, lambda_dnm=1.0, lambda_eik=1.0, lambda_fd=0.0)
    from oracle.c_oracle import _spec, _loss, _run
    s = _spec(None, "sphere", [0, 0, 0, 0.5, 2.0])
    out, loss, _ = _run(s, None, x, np.array([1, 1], np.uint8), 1e-2, _loss(cfg, (2, 0, 2)), 0,
                        np.arange(2, dtype=np.int64), None, False, 0, 1)
    assert loss[0] == pytest.approx(0.1, abs=1e-12)
    assert loss[2] == pytest.approx(1.0, abs=1e-12)
    out, loss, _ = _run(s, None, np.array([[0.525, 0, 0]]), np.array([0], np.uint8), 1e-2,
                        _loss(cfg, (0, 1, 1)), 0, np.arange(1, dtype=np.int64), None, False, 0, 1)
    assert loss[1] == pytest.approx(math.exp(-5), rel=1e-12)
    c = make_config("c1", 32, 32)
    base = dict(kind="ncr", denom="paper", w_dm=0.0, lambda_dnm=0.0, lambda_eik=0.0, lambda_fd=0.0,
                alpha_dnm=100.0, fd_form="abs", denom_pow=4, eps_grad=1e-6)
    parts = []
    for k in ("w_dm", "lambda_dnm", "lambda_eik", "lambda_fd"):
        parts.append(c_oracle_step(c["spec"], c["params"], c["x"], 32, c["h"], dict(base, **{k: 1.0}),
                                   frame_seed=3)["loss"][4])
    w = dict(base, w_dm=2.0, lambda_dnm=3.0, lambda_eik=5.0, lambda_fd=7.0)
    tot = c_oracle_step(c["spec"], c["params"], c["x"], 32, c["h"], w, frame_seed=3)["loss"][4]
    assert tot == pytest.approx(2 * parts[0] + 3 * parts[1] + 5 * parts[2] + 7 * parts[3], rel=1e-13)


LOSS_VARIANTS = [
    dict(kind="ncr", denom="paper", w_dm=1.0, lambda_dnm=100.0, lambda_eik=50.0, lambda_fd=1.0, fd_form="abs"),
    dict(kind="ncr", denom="grad", w_dm=0.0, lambda_dnm=0.0, lambda_eik=0.0, lambda_fd=1.0, fd_form="abs"),
    dict(kind="nsh", denom="one", w_dm=1.0, lambda_dnm=0.0, lambda_eik=50.0, lambda_fd=1.0, fd_form="square"),
]
NETS = [("softplus", [3, 8, 8, 1], -1, 30.0, 30.0), ("sine", [3, 8, 8, 1], -1, 3.0, 2.0),
        ("softplus", [3, 6, 5, 6, 1], 2, 30.0, 30.0)]


@pytest.mark.parametrize("net", range(len(NETS)))
@pytest.mark.parametrize("variant", range(len(LOSS_VARIANTS)))
def test_c_weight_gradient_brute_force(net, variant):
    """Central FD of the C oracle's fp64 total loss over EVERY parameter of tiny nets (softplus,
    sine with omega0_first != omega0_hidden, a skip-layer net), frames and mask frozen (SURVEY
    §8c item 8), matches the hand-derived reverse sweep: relL2 < 1e-6."""
    act, widths, skip, om1, om2 = NETS[net]
    spec = mlp_spec(widths, act, beta=10.0, omega0_first=om1, omega0_hidden=om2, skip_at=skip)
    P = init_params(spec, "siren" if act == "sine" else "xavier", 3 + variant).astype(np.float64)
    if act == "softplus":
        P += np.random.default_rng(30 + net).normal(0, 0.05, P.size)  # nonzero biases
    cfg = dict(LOSS_VARIANTS[variant], alpha_dnm=100.0, denom_pow=4, eps_grad=1e-6)
    x = np.random.default_rng(12 + variant).uniform(-0.8, 0.8, (20, 3))
    h = 2e-2
    ref = c_oracle_step(spec, P, x, 10, h, cfg, frame_seed=77, promote=False)
    assert ref["mask"].all()
    frames = (ref["u"], ref["v"])

    def loss_at(p):
        return c_oracle_step(spec, p, x, 10, h, cfg, frames=frames, promote=False, need_grad=False)["loss"][4]

    assert loss_at(P) == pytest.approx(ref["loss"][4], rel=1e-14)
    fd = np.empty(P.size)
    for i in range(P.size):
        e = 1e-6 * max(1.0, abs(P[i]))
        Pp, Pm = P.copy(), P.copy()
        Pp[i] += e
        Pm[i] -= e
        fd[i] = (loss_at(Pp) - loss_at(Pm)) / (2 * e)
    g = ref["grad"]
    assert np.linalg.norm(fd - g) / np.linalg.norm(g) < 1e-6


def test_c_output_bias_invariance():
    """f_uu, f_vv, f_uv and g do not depend on b_L: dL_fd/db_L = dL_eik/db_L = 0 exactly (App.B)."""
    spec = mlp_spec([3, 8, 8, 1], "sine", omega0_first=30.0, omega0_hidden=15.0)
    params = init_params(spec, "siren", 9)
    x = np.random.default_rng(13).uniform(-0.8, 0.8, (16, 3)).astype(np.float32)
    cfg = dict(kind="ncr", denom="grad", w_dm=0.0, lambda_dnm=0.0, lambda_eik=50.0, lambda_fd=1.0,
               fd_form="abs", alpha_dnm=100.0, denom_pow=4, eps_grad=1e-6)
    o = c_oracle_step(spec, params, x, 8, 1e-2, cfg, frame_seed=3)
    assert o["grad"][-1] == 0.0


def test_c_degenerate_mask_counts_and_flags():
    """Centres with |g| < eps_grad are masked: u = v = 0, entries / D / K = 0, no
    FD loss, counted in loss[5]; the torch oracle agrees on the count and the gradient."""
    c = make_config("c1", 40, 40)
    cfg = dict(c["loss"], w_dm=1.0, lambda_eik=50.0)
    gn = np.linalg.norm(c_oracle_eval(c["spec"], c["params"], c["x"], 40, c["h"])["g"], axis=1)
    srt = np.sort(gn)
    j = int(np.argmax(np.diff(srt[20:60]))) + 20
    eps = 0.5 * (srt[j] + srt[j + 1])
    cfg["eps_grad"] = eps
    o = c_oracle_step(c["spec"], c["params"], c["x"], 40, c["h"], cfg, frame_seed=5)
    m = gn >= eps
    assert np.array_equal(o["mask"], m) and o["loss"][5] == float((~m).sum()) > 0
    assert np.all(o["u"][~m] == 0) and np.all(o["K"][~m] == 0) and np.all(o["fuu"][~m] == 0)
    t = oracle_step(c["spec"], c["params"], c["x"], 40, c["h"], cfg, frame_seed=5)
    assert t["loss"][5] == o["loss"][5]
    assert np.linalg.norm(t["grad"] - o["grad"]) <= 1e-9 * np.linalg.norm(t["grad"])

# ----------------------------------------------------------------------------- the two oracles agree


CROSS = [("c1", 24, 24, None), ("c1", 20, 17, loss_cfg("ncr", "grad", w_dm=1, lambda_dnm=100, lambda_eik=50)),
         ("c1", 16, 16, loss_cfg("nsh", "one", w_dm=1, lambda_dnm=100, lambda_eik=50, fd_form="square")),
         ("c2", 8, 8, None), ("c3", 2, 2, None), ("c4", 6, 5, None)]


@pytest.mark.parametrize("case", range(len(CROSS)))
def test_c_and_torch_oracles_agree(case):
    """Two independent fp64 implementations (plain C reverse sweeps; PyTorch autograd) of the
    same definitions agree far below every GPU tolerance: entries 1e-9 (1 + |ref|), loss 1e-9
    relative, gradient relL2 1e-8."""
    name, ns, nu, ls = CROSS[case]
    c = make_config(name, ns, nu)
    if ls is not None:
        c["loss"] = ls
    a = oracle_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    b = c_oracle_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    assert np.array_equal(a["mask"], b["mask"])
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "u", "v"):
        assert np.max(np.abs(a[k] - b[k]) / (1 + np.abs(a[k]))) < 1e-9, k
    assert np.max(np.abs(a["K"] - b["K"]) / (1 + np.abs(a["K"]))) < 1e-8
    nz = a["loss"][:5] != 0
    assert np.all(np.abs(a["loss"][:5][nz] - b["loss"][:5][nz]) / np.abs(a["loss"][:5][nz]) < 1e-9)
    assert np.linalg.norm(a["grad"] - b["grad"]) / np.linalg.norm(a["grad"]) < 1e-8


def test_c_hessian_matches_definition():
    """The 19-point world-axis Hessian (NEXT-4) of the C oracle equals the torch oracle's on the C2
    net (the same definition, two implementations)."""
    from oracle import oracle_hessian
    c = make_config("c2", 6, 6)
    f, H = c_oracle_hessian(c["spec"], c["params"], c["x"], 1e-2)
    f2, H2 = oracle_hessian(c["spec"], c["params"], c["x"], 1e-2)
    assert np.allclose(f, f2, rtol=1e-13, atol=1e-15) and np.max(np.abs(H - H2) / (1 + np.abs(H2))) < 1e-9
