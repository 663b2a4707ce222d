"""fp64 / exact-integer CPU oracle of the training-iteration steps around the FD step
(SURVEY §8f NEXT-1).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Written from the paper and the documented
generator contract (include/fdsdf.h fdsdf_sample / fdsdf_adam), not from the CUDA code:

 * sample_batch: the per-iteration batch of PAPER.md §4 "Datasets" ("we sample 30k
   surface points; 20k are used per iteration, with 20k off-surface samples drawn uniformly in
   the bounding box").  Rows [0, n_pick): pool rows pi(0..n_pick-1), pi a keyed pseudo-random
   permutation of [0, n_pool) -- a 4-round balanced Feistel network on 2b bits
   (b = ceil(bits(n_pool - 1) / 2)), round function mix64(key + (r+1)*gamma + R) & mask,
   cycle-walked into range, key = mix64(seed ^ ((iteration+1)*gamma2)); sampling WITHOUT
   replacement follows because pi is a bijection.  Rows [n_pick, ...): uniform in
   [-half, half]^3, U = (mix64(seed2 + ((iteration*n_uniform + j)*3 + d + 1)*gamma) >> 11)
   * 2^-53, seed2 = mix64(~seed), coordinate = half*(2U - 1) in fp64 rounded to fp32.
   Plain python integers; a loop per row.
 * adam_step: the Adam update of P:L153 ("Adam optimizer (5e-5)") in its standard
   bias-corrected form (Kingma & Ba), fp64 on numpy arrays.

Parity unpinned: none (tests/test_train_oracle.py pins the Feistel bijection by brute force,
the box sampler by its moments and bounds, and Adam by closed forms).
"""
from __future__ import annotations

import numpy as np

from .fdsdf_oracle import splitmix64

__all__ = ["feistel_perm", "sample_indices", "sample_batch", "adam_step"]

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_GAMMA2 = 0xD1B54A32D192ED03


def _half_bits(n_pool):
    bits = 1
    while bits < 62 and ((n_pool - 1) >> bits) > 0:
        bits += 1
    return (bits + 1) // 2


def feistel_perm(x, key, b):
    """One pass of the 4-round balanced Feistel network on 2b-bit integers."""
    mask = (1 << b) - 1
    L, R = x >> b, x & mask
    for r in range(4):
        L, R = R, L ^ (splitmix64((key + (r + 1) * _GAMMA + R) & _M64) & mask)
    return (L << b) | R


def sample_indices(n_pool, n_pick, seed, iteration):
    """Pool indices of the n_pick surface rows of iteration `iteration`."""
    key = splitmix64((int(seed) ^ (((int(iteration) + 1) * _GAMMA2) & _M64)) & _M64)
    b = _half_bits(n_pool)
    out = np.empty(n_pick, np.int64)
    for j in range(n_pick):
        x = j
        while True:
            x = feistel_perm(x, key, b)
            if x < n_pool:
                break
        out[j] = x
    return out


def sample_batch(pool, n_pick, half, n_uniform, seed, iteration):
    """[n_pick + n_uniform, 3] fp32: distinct pool rows, then uniform box points."""
    pool = np.asarray(pool, np.float32).reshape(-1, 3)
    idx = sample_indices(len(pool), n_pick, seed, iteration) if n_pick else np.zeros(0, np.int64)
    seed2 = splitmix64((~int(seed)) & _M64)
    half = float(np.float32(half))  # the C ABI takes box_half as fp32
    box = np.empty((n_uniform, 3), np.float32)
    for j in range(n_uniform):
        for d in range(3):
            k = splitmix64((seed2 + ((int(iteration) * n_uniform + j) * 3 + d + 1) * _GAMMA) & _M64)
            U = float(k >> 11) * 2.0 ** -53
            box[j, d] = np.float32(float(half) * (2.0 * U - 1.0))
    return np.concatenate([pool[idx], box], 0)


def adam_step(p, g, m, v, t, lr=5e-5, b1=0.9, b2=0.999, eps=1e-8):
    """Bias-corrected Adam in fp64; returns (p, m, v) new arrays.
    Non-finite gradient entries leave their parameter and moments unchanged."""
    p, g, m, v = (np.asarray(a, np.float64) for a in (p, g, m, v))
    ok = np.isfinite(g)
    gz = np.where(ok, g, 0.0)
    m2 = np.where(ok, b1 * m + (1 - b1) * gz, m)
    v2 = np.where(ok, b2 * v + (1 - b2) * gz * gz, v)
    mh = m2 / (1 - b1 ** t)
    vh = v2 / (1 - b2 ** t)
    p2 = np.where(ok, p - lr * mh / (np.sqrt(vh) + eps), p)
    return p2, m2, v2
