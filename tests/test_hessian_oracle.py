"""Pins of the 19-point world-axis FD Hessian of the oracle (oracle.fd_hessian /
oracle_hessian, the P:L83-91 stencil formulas with (u, v) = (e_i, e_j))
against closed forms, invariants and the textbook convergence order -- not against itself."""
import math

import numpy as np
import torch

from harness import make_config
from oracle import fd_hessian, hessian_at, oracle_hessian, sdf, unflatten

F64 = torch.float64
IDX = [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]


def _t(a):
    return torch.as_tensor(np.asarray(a, np.float64), dtype=F64)


def _sym(H6):
    H = np.zeros(H6.shape[:-1] + (3, 3))
    for k, (i, j) in enumerate(IDX):
        H[..., i, j] = H[..., j, i] = H6[..., k]
    return H


def test_quadratic_exact_for_any_h():
    """f = 1/2 x^T A x + b.x + c: the 19-point stencil returns A exactly (third and fourth
    derivatives vanish), up to rounding of f / h^2."""
    rng = np.random.default_rng(21)
    A = rng.normal(size=(3, 3))
    A = A + A.T
    b = rng.normal(size=3)
    field = lambda x: 0.5 * ((x @ _t(A)) * x).sum(1) + x @ _t(b) - 0.3  # noqa: E731
    x0 = rng.uniform(-1, 1, (40, 3))
    for h in (1e-1, 1e-2, 1e-3):
        H = _sym(fd_hessian(field, _t(x0), h).numpy())
        tol = 64 * 2.2e-16 * 10.0 / h ** 2
        assert np.abs(H - A[None]).max() < tol, h


def test_sphere_on_axis_closed_form():
    """f = |x| - r at x0 = rho e_k: the axial second difference is 0 (f is linear along
    e_k there), the transverse ones are 2 (sqrt(rho^2 + h^2) - rho) / h^2 =
    2 / (sqrt(rho^2 + h^2) + rho), and every mixed entry vanishes by the y -> -y symmetry."""
    r = 0.5
    field = lambda x: torch.linalg.vector_norm(x, dim=1) - r  # noqa: E731
    for k in range(3):
        for rho in (0.5, 0.8):
            x0 = np.zeros((1, 3))
            x0[0, k] = rho
            for h in (2e-2, 5e-3):
                H = _sym(fd_hessian(field, _t(x0), h).numpy())[0]
                want = 2.0 / (math.sqrt(rho * rho + h * h) + rho)
                tol = 1e-15 / h ** 2 * 10
                for i in range(3):
                    assert abs(H[i, i] - (0.0 if i == k else want)) < tol
                    for j in range(3):
                        if i != j:
                            assert abs(H[i, j]) < tol


def test_axis_permutation_covariance():
    """Relabelling the coordinates permutes the Hessian: for f'(x) = f(P x) with a
    permutation P, H'(x0) = P^T H(P x0) P entry by entry (the stencil maps onto itself)."""
    rng = np.random.default_rng(22)
    field = lambda x: torch.sin(3 * x[:, 0] + x[:, 1] ** 2) * torch.exp(0.5 * x[:, 2]) + x[:, 0] * x[:, 2]  # noqa: E731
    P = np.eye(3)[[2, 0, 1]]
    fieldp = lambda x: field(x @ _t(P).T)  # noqa: E731
    x0 = rng.uniform(-0.7, 0.7, (20, 3))
    h = 1e-2
    H = _sym(fd_hessian(field, _t(x0 @ P.T), h).numpy())
    Hp = _sym(fd_hessian(fieldp, _t(x0), h).numpy())
    assert np.abs(Hp - np.einsum("ai,nab,bj->nij", P, H, P)).max() < 1e-9


def test_converges_to_mlp_hessian_order_two():
    """On the C1 / C2 networks the FD Hessian approaches the analytic Hessian of the MLP
    at O(h^2): err(h) / err(h/2) in [3.5, 4.5] (the standard central-difference order,
    P:L92 / appendix)."""
    for name in ("c1", "c2"):
        c = make_config(name, 8, 8)
        spec, params = c["spec"], c["params"].astype(np.float64)
        layers = unflatten(spec, _t(params))
        field = lambda x: sdf(spec, layers, x)  # noqa: E731
        ratios = []
        for x0 in c["x"][:10].astype(np.float64):
            _, Hx = hessian_at(field, x0)
            errs = []
            for h in (2e-2, 1e-2, 5e-3, 2.5e-3):
                Hf = _sym(fd_hessian(field, _t([x0]), h).numpy())[0]
                errs.append(np.abs(Hf - Hx.numpy()).max())
            ratios += [errs[i] / errs[i + 1] for i in range(3)]
        ratios = np.array(ratios)
        assert 3.5 <= np.median(ratios) <= 4.5, (name, ratios)
        assert np.mean((ratios >= 3.5) & (ratios <= 4.5)) >= 0.8, (name, ratios)


def test_oracle_hessian_promotes_fp32_inputs():
    """oracle_hessian evaluates at the fp32 centres and h promoted exactly:
    its f equals sdf at those points and its H equals fd_hessian with h = (double)(float)h."""
    c = make_config("c1", 6, 6)
    f, H = oracle_hessian(c["spec"], c["params"], c["x"], 1e-2)
    layers = unflatten(c["spec"], _t(c["params"].astype(np.float32)))
    field = lambda x: sdf(c["spec"], layers, x)  # noqa: E731
    x0 = _t(c["x"].astype(np.float32))
    assert np.array_equal(f, field(x0).numpy())
    assert np.array_equal(H, fd_hessian(field, x0, float(np.float32(1e-2))).numpy())
