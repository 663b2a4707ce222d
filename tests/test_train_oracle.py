"""Pins of the training-iteration oracle (oracle/train_oracle.py) against
what mathematics fixes -- no GPU.

 * the keyed Feistel map is a bijection of [0, 2^(2b)) (brute force), so the surface subset
   is sampling WITHOUT replacement ("20k are used per iteration");
 * the box sampler lies in [-half, half]^3 and has the moments of U(-half, half)
   (mean 0, variance half^2/3), independent across coordinates;
 * Adam: for a constant gradient g from a zero state every bias-corrected step moves the
   parameter by exactly -lr*g/(|g|+eps) (closed form); with beta1 = beta2 = 0 the update is
   -lr*g/(|g|+eps) for any gradient sequence; non-finite entries are skipped.
"""
import numpy as np
import pytest

from oracle.train_oracle import adam_step, feistel_perm, sample_batch, sample_indices


@pytest.mark.parametrize("b", [1, 2, 3, 5])
def test_feistel_is_a_bijection(b):
    for key in (0, 1, 0xDEADBEEF12345678):
        img = sorted(feistel_perm(x, key, b) for x in range(1 << (2 * b)))
        assert img == list(range(1 << (2 * b)))


@pytest.mark.parametrize("n_pool,n_pick", [(1, 1), (7, 7), (30, 20), (1000, 667), (3000, 2000)])
def test_subset_without_replacement(n_pool, n_pick):
    idx = sample_indices(n_pool, n_pick, seed=11, iteration=3)
    assert len(idx) == n_pick and len(set(idx.tolist())) == n_pick
    assert idx.min() >= 0 and idx.max() < n_pool
    if n_pick == n_pool:
        assert sorted(idx.tolist()) == list(range(n_pool))


def test_subsets_change_per_iteration_and_cover_pool():
    n_pool, n_pick = 300, 200
    seen = np.zeros(n_pool, int)
    a = sample_indices(n_pool, n_pick, 5, 0)
    b = sample_indices(n_pool, n_pick, 5, 1)
    assert not np.array_equal(np.sort(a), np.sort(b))
    for it in range(60):
        seen[sample_indices(n_pool, n_pick, 5, it)] += 1
    # each pool row is picked with probability 2/3 per iteration: 40 +- 4 sigma over 60 draws
    assert seen.min() > 40 - 4 * np.sqrt(60 * 2 / 9) and seen.max() < 40 + 4 * np.sqrt(60 * 2 / 9)


def test_box_points_moments():
    half = 1.1
    pts = sample_batch(np.zeros((1, 3), np.float32), 0, half, 20000, seed=3, iteration=7)
    assert pts.shape == (20000, 3) and pts.dtype == np.float32
    assert np.all(np.abs(pts) <= half)
    m = pts.mean(0)
    var = pts.var(0)
    se = half / np.sqrt(3 * 20000)
    assert np.all(np.abs(m) < 5 * se)
    assert np.all(np.abs(var - half ** 2 / 3) < 0.02 * half ** 2 / 3 * 3)
    c = np.corrcoef(pts.T)
    assert np.all(np.abs(c[np.triu_indices(3, 1)]) < 0.05)


def test_batch_layout_rows():
    pool = np.arange(30 * 3, dtype=np.float32).reshape(30, 3)
    x = sample_batch(pool, 20, 1.0, 5, seed=1, iteration=0)
    idx = sample_indices(30, 20, 1, 0)
    assert np.array_equal(x[:20], pool[idx])
    assert np.all(np.abs(x[20:]) <= 1.0)


def test_adam_constant_gradient_closed_form():
    rng = np.random.default_rng(0)
    p0 = rng.standard_normal(50)
    g = rng.standard_normal(50) * np.exp(rng.uniform(-6, 2, 50))
    lr, eps = 5e-5, 1e-8
    p, m, v = p0.copy(), np.zeros(50), np.zeros(50)
    for t in range(1, 8):
        p, m, v = adam_step(p, g, m, v, t, lr=lr, eps=eps)
        np.testing.assert_allclose(p, p0 - t * lr * g / (np.abs(g) + eps), rtol=0, atol=1e-15)


def test_adam_memoryless_betas_zero():
    rng = np.random.default_rng(1)
    p, m, v = rng.standard_normal(20), np.zeros(20), np.zeros(20)
    for t in range(1, 5):
        g = rng.standard_normal(20)
        p_new, m, v = adam_step(p, g, m, v, t, lr=1e-3, b1=0.0, b2=0.0, eps=1e-8)
        np.testing.assert_allclose(p_new, p - 1e-3 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
        p = p_new


def test_adam_skips_nonfinite():
    p, g = np.ones(4), np.array([1.0, np.nan, np.inf, -2.0])
    p2, m2, v2 = adam_step(p, g, np.zeros(4), np.zeros(4), 1)
    assert p2[1] == 1.0 and p2[2] == 1.0 and m2[1] == 0.0 and v2[2] == 0.0
    assert p2[0] < 1.0 and p2[3] > 1.0
