"""tcgen05 contraction core (csrc/tc.cuh) through fdsdf_selftest_mma: descriptor / swizzle /
TMEM-mapping correctness and the accuracy of the bf16 piece schemes.

Reference: the same GEMM in fp64 numpy.  bf16x6 must be fp32-accurate (a few fp32 ulps of the
sum of |products| per entry, within a small factor of a sequential fp32 chain); plain bf16 (1 product) must NOT be, which shows the pieces are
really used."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


def _run(M, N, K, nprod, seed=0, structured=False, mn=0):
    from paper_2511_08980_b200.fdsdf import fdsdf_selftest_mma
    rng = np.random.default_rng(seed)
    if structured:
        # distinct value per (row, k) so any permutation of rows / k chunks shows up
        W = (np.arange(M)[:, None] * 1.0 + np.arange(K)[None, :] * 1e-3).astype(np.float32)
        B = np.zeros((N, K), np.float32)
        B[np.arange(N), (np.arange(N) * 7) % K] = 1.0
    else:
        W = rng.standard_normal((M, K)).astype(np.float32)
        B = (rng.standard_normal((N, K)) * np.exp(rng.uniform(-8, 0, (N, 1)))).astype(np.float32)
    D = fdsdf_selftest_mma(torch.from_numpy(W).cuda(), torch.from_numpy(B).cuda(), nprod, mn)
    torch.cuda.synchronize()
    ref = W.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(W.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    return D.cpu().numpy().astype(np.float64), ref, scale


@pytest.mark.parametrize("M,N,K", [(128, 64, 256), (256, 64, 256), (256, 80, 256), (128, 128, 512),
                                   (256, 256, 64), (128, 16, 128)])
def test_mma_layout_structured(M, N, K):
    D, ref, _ = _run(M, N, K, 6, structured=True)
    assert np.array_equal(D, ref.astype(np.float32).astype(np.float64)) or np.max(np.abs(D - ref)) < 1e-3


@pytest.mark.parametrize("M,N,K", [(256, 64, 256), (128, 80, 512), (256, 256, 128)])
def test_mma_bf16x6_is_fp32_accurate(M, N, K):
    D, ref, scale = _run(M, N, K, 6, seed=M + N + K)
    err = np.max(np.abs(D - ref) / (scale * 2.0 ** -24))
    # the same contraction as a sequential fp32 FFMA chain (what the FFMA kernels do)
    rng = np.random.default_rng(M + N + K)
    W = rng.standard_normal((M, K)).astype(np.float32)
    B = (rng.standard_normal((N, K)) * np.exp(rng.uniform(-8, 0, (N, 1)))).astype(np.float32)
    seq = np.cumsum(W[:, None, :] * B[None, :, :], axis=-1, dtype=np.float32)[..., -1].astype(np.float64)
    err32 = np.max(np.abs(seq - ref) / (scale * 2.0 ** -24))
    print(f"bf16x6 err {err:.2f} vs sequential fp32 {err32:.2f} (fp32 ulps of sum|ab|)")
    # measured on B200: ~14 ulps (the tensor core's fp32 accumulation is not round-to-nearest);
    # ~4x a sequential fp32 chain, i.e. ~1e-6 relative to sum|ab| -- far inside the 1e-4 gates
    assert err <= max(24.0, 6.0 * err32)
    D1, _, _ = _run(M, N, K, 1, seed=M + N + K)
    err1 = np.max(np.abs(D1 - ref) / (scale * 2.0 ** -24))
    print("bf16x1 err:", err1)
    assert err1 > 100.0


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (128, 64, 64), (256, 128, 256), (128, 192, 128),
                                   (128, 80, 128), (256, 160, 128), (128, 240, 64), (128, 16, 64)])
def test_mma_mn_major(M, N, K):
    """MN-major operands (LBO = stride between swizzle atoms along M/N, SBO = along K), the
    layout of the weight-gradient kernel and of the forward kernels' B operand; N not a multiple
    of the 64-column swizzle atom (a partial last atom) is the backward's N = 80 / 160."""
    D, ref, scale = _run(M, N, K, 6, seed=7, mn=1)
    err = np.max(np.abs(D - ref) / (scale * 2.0 ** -24))
    print("mn-major", M, N, K, "err ulps", err)
    assert err <= 24.0
    Ds, refs, _ = _run(M, N, K, 6, structured=True, mn=1)
    assert np.max(np.abs(Ds - refs)) < 1e-3


@pytest.mark.parametrize("N,K", [(64, 128), (128, 256), (256, 64), (96, 192)])
def test_mma_cta_pair(N, K):
    """cta_group::2 (M = 256 over a CTA pair, B split by columns between the pair)."""
    from paper_2511_08980_b200.fdsdf import fdsdf_selftest_mma_pair
    rng = np.random.default_rng(N + K)
    W = rng.standard_normal((256, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    D = fdsdf_selftest_mma_pair(torch.from_numpy(W).cuda(), torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    D = D.cpu().numpy().astype(np.float64)
    ref = W.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(W.astype(np.float64)) @ np.abs(B.astype(np.float64)).T
    err = np.max(np.abs(D - ref) / (scale * 2.0 ** -24))
    print("pair", N, K, "err ulps", err)
    assert err <= 24.0
