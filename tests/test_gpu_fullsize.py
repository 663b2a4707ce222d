"""Parity at BASELINE.json's full sizes in the launch configuration bench.py times (the default
tensor-core path, one CTA per SM over all tiles).

 * C2 (bench workload, 40k centres): every row's f, grad f, FD entries, D, K against the oracle
   (GIVEN frames exported by the GPU), and the step's loss / weight gradient against the oracle
   on the full batch.
 * C5 (data-parallel shard, 200k centres): eval entries on 3000 sampled rows; the step's loss and
   gradient against the oracle accumulated over 20k-row chunks with the global counts (the
   loss and gradient are sums of per-centre terms).
 * C5e (the eval sweep's 10^6-centre size, eval-only context): 512 sampled rows against the C oracle.
 * C4 h sweep (2e-2 .. 2.5e-3): BJ fixes the 1e-4 gate at h = 1e-2; the difference form
    keeps every entry inside that same gate at every h of the sweep (measured
   worst: 0.29 of the gate at h = 2.5e-3), so the test applies it unscaled.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config  # noqa: E402
from gpu_util import ref_step, ref_eval  # noqa: E402
from oracle import oracle_step, oracle_eval  # noqa: E402  (batched torch fp64 oracle for the 200k-centre C5 check)
from gpu_util import compare_eval, gpu_eval, per_tensor_grad_errors, LOSS_RTOL, GRAD_RTOL  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


def _model(spec, n, eval_only=False):
    from paper_2511_08980_b200 import FDSDF
    m = FDSDF(spec, 0, max_centers=n, eval_only=eval_only)
    assert m.path == "tensor"
    return m


def _check_step(c, n_chunk=None, step_fn=ref_step):
    n = len(c["x"])
    m = _model(c["spec"], n)
    ev = gpu_eval(m, c, denom=c["loss"]["denom"])
    grad, loss = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    fr = ev["frames"]
    counts = (c["n_surface"], n - c["n_surface"], n)
    n_chunk = n_chunk or n
    ol, og = np.zeros(8), 0.0
    for s in range(0, n, n_chunk):
        e = min(n, s + n_chunk)
        surf = np.arange(s, e) < c["n_surface"]
        o = step_fn(c["spec"], c["params"], c["x"][s:e], 0, c["h"], c["loss"], frames=(fr[s:e, :3], fr[s:e, 3:]),
                        counts=counts, surface_mask=surf, gidx=range(s, e))
        ol[:6] += o["loss"][:6]
        og = og + o["grad"]
    # each chunk's terms are already divided by the global counts: the chunk sums are the totals
    lerr = np.abs(loss[:5] - ol[:5]) / np.maximum(np.abs(ol[:5]), 1e-30)
    gerr = per_tensor_grad_errors(c["spec"], grad, og)
    print(c["name"], n, "loss", loss[:5], "lerr", lerr, "gerr max", gerr.max())
    for i in range(5):
        if ol[i] != 0:
            assert lerr[i] <= LOSS_RTOL, (i, lerr)
    assert loss[5] == ol[5]
    assert np.all(gerr <= GRAD_RTOL), gerr
    return ev


def test_c2_full_eval_and_step():
    c = make_config("c2")
    ev = _check_step(c)
    o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"],
                    frames=(ev["frames"][:, :3], ev["frames"][:, 3:]))
    err = compare_eval(ev, o)
    print("c2 full eval", {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    assert err["mask"] == 0


def test_c5_full_step_chunked_oracle():
    """C5 (200k centres): checked against the batched PyTorch fp64 oracle (the C oracle, ~6 ms per
    centre on one core, would need ~20 CPU-minutes; both oracles are pinned and agree to 1e-9,
    tests/test_c_oracle_pins.py)."""
    c = make_config("c5")
    ev = _check_step(c, n_chunk=20_000, step_fn=oracle_step)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(len(c["x"]), 3000, replace=False))
    o = oracle_eval(c["spec"], c["params"], c["x"][rows], 0, c["h"],
                    frames=(ev["frames"][rows, :3], ev["frames"][rows, 3:]))
    sub = {k: v[rows] for k, v in ev.items()}
    # the PAPER denominator policy depends on the role: recompute the oracle's K on these rows
    # with the rows' own roles
    o2 = oracle_step(c["spec"], c["params"], c["x"][rows], 0, c["h"],
                     dict(c["loss"], w_dm=0.0, lambda_dnm=0.0, lambda_eik=0.0, lambda_fd=0.0),
                     frames=(ev["frames"][rows, :3], ev["frames"][rows, 3:]), need_grad=False,
                     surface_mask=rows < c["n_surface"], gidx=rows)
    o["K"] = o2["K"]
    err = compare_eval(sub, o)
    print("c5 sampled eval", {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)


@pytest.mark.parametrize("h", [2e-2, 1e-2, 5e-3, 2.5e-3])
def test_c4_h_sweep(h):
    c = make_config("c4", 600, 600, h=h)
    m = _model(c["spec"], len(c["x"]), eval_only=True)
    g = gpu_eval(m, c)
    o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"],
                    frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    err = compare_eval(g, o)
    print("c4 h", h, {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    assert err["mask"] == 0


@pytest.mark.parametrize("path", [None, "ffma"])
def test_c3_full_size(path):
    """C3 (softplus 3->512x8->1 with the skip layer, 100k centres; default = the hybrid path:
    tensor-core forward with the skip input and weight gradient, FFMA backward; and the FFMA
    path):
    f, grad f, FD entries, D, K on 400 sampled rows of the full-size eval against the oracle
    (GIVEN frames exported by the GPU); the full-size step is finite and bitwise reproducible.
    The oracle cannot afford the full C3 step (~11 TFLOP in fp64 on the host), so the step's
    loss / gradient parity is covered at C3 sizes in test_gpu_parity.py."""
    import time
    from paper_2511_08980_b200 import FDSDF
    c = make_config("c3")
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n, path=path)
    assert m.path == ("hybrid" if path is None else "ffma"), m.path
    ev = gpu_eval(m, c, denom=c["loss"]["denom"])
    rng = np.random.default_rng(33)
    idx = np.sort(rng.choice(n, 400, replace=False))
    sub = {k: v[idx] for k, v in ev.items()}
    fr = sub["frames"]
    surf = idx < c["n_surface"]
    o = ref_eval(c["spec"], c["params"], c["x"][idx], int(surf.sum()), c["h"], frames=(fr[:, :3], fr[:, 3:]),
                    denom=c["loss"]["denom"])
    # oracle_eval assumes a surface prefix: the sampled rows are sorted, so surface rows come first
    err = compare_eval(sub, o)
    print("c3 full-size sampled eval errors", {k: float(v) for k, v in err.items()},
          "max |df|", float(np.abs(sub["f"] - o["f"]).max()), "max |f|", float(np.abs(o["f"]).max()))
    assert all(err[k] <= 1.0 for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K")), err
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g1, l1 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    g1, l1 = g1.cpu().numpy(), l1.cpu().numpy()
    g2, l2 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    print(f"c3 full-size step [{m.path}] {dt * 1e3:.1f} ms (wall, 1st call), loss {l1[:5]}")
    assert np.isfinite(l1).all() and np.isfinite(g1).all()
    assert np.array_equal(g1, g2.cpu().numpy()) and np.array_equal(l1, l2.cpu().numpy())
    m.close()


def test_c3_step_parity_first_rows():
    """C3's loss (FD-NSH, (1, 100, 50, 1), den 1, h = 1e-2) and weight gradient on the first 1024
    surface + 1024 uniform rows of the C3 batch against the fp64 C oracle, on the
    default (hybrid) path and the FFMA path, with the frames the GPU drew (GIVEN mode for both
    GPU steps and the oracle)."""
    from paper_2511_08980_b200 import FDSDF
    c = make_config("c3", 1024, 1024)
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n)
    assert m.path == "hybrid", m.path
    ev = gpu_eval(m, c, denom=c["loss"]["denom"])
    fr = ev["frames"]
    o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frames=(fr[:, :3], fr[:, 3:]))
    for path in (None, "ffma"):
        mm = m if path is None else FDSDF(c["spec"], 0, max_centers=n, path=path)
        grad, loss = mm.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frames=fr)
        grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
        lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
        gerr = per_tensor_grad_errors(c["spec"], grad, o["grad"])
        print("c3 first rows", mm.path, "lerr", lerr, "gerr max", gerr.max())
        assert np.all(lerr[o["loss"][:5] != 0] <= LOSS_RTOL), lerr
        assert loss[5] == o["loss"][5]
        assert np.all(gerr <= GRAD_RTOL), gerr
        if path is not None:
            mm.close()
    m.close()


def test_c5e_eval_sweep_size_sampled():
    """C5e (SURVEY §8d's eval target, the bench's `eval_sweep`): fdsdf_eval over 10^6 centres on an
    eval-only context, as bench.py runs it (C2's network, half CSG surface / half uniform rows,
    h = 5e-3) -- 512 sampled rows (the first and the last tile included) against the C oracle with
    the GPU's exported frames; the frames themselves must be orthonormal, right-handed and
    tangent to the oracle's gradient on every sampled row, and every output finite on all rows."""
    from harness import csg_surface, uniform_box
    c = make_config("c2", 64, 64)  # network, parameters, h of the sweep; the points are replaced below
    n = 1_000_000
    x = np.concatenate([csg_surface(n // 2, 3, 7), uniform_box(n - n // 2, 1.1, 8)]).astype(np.float32)
    ns = n // 2
    m = _model(c["spec"], n, eval_only=True)
    o = m.eval(c["params"], x, ns, c["h"], frame_seed=0)
    ev = {k: v.cpu().numpy() for k, v in o.items()}
    for k in ("f", "g", "hess", "D", "K", "frames"):
        assert np.isfinite(ev[k]).all(), k
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([np.arange(8), np.arange(n - 8, n), [ns - 1, ns], rng.choice(n, 494, replace=False)]))
    sub = {k: v[idx] for k, v in ev.items()}
    fr = sub["frames"]
    surf = idx < ns
    ref = ref_eval(c["spec"], c["params"], x[idx], int(surf.sum()), c["h"], frames=(fr[:, :3], fr[:, 3:]))
    err = compare_eval(sub, ref)
    print("c5e 1e6-centre sampled eval errors", {k: float(v) for k, v in err.items()})
    assert all(err[k] <= 1.0 for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K")), err
    assert err["mask"] == 0
    # the exported frames: orthonormal, right-handed, tangent to the oracle's normal
    u, v = fr[:, :3].astype(np.float64), fr[:, 3:].astype(np.float64)
    nrm = ref["g"] / np.linalg.norm(ref["g"], axis=1, keepdims=True)
    assert np.abs(np.linalg.norm(u, axis=1) - 1).max() < 1e-5 and np.abs(np.linalg.norm(v, axis=1) - 1).max() < 1e-5
    assert np.abs((u * v).sum(1)).max() < 1e-5
    assert np.abs((u * nrm).sum(1)).max() < 1e-4 and np.abs((v * nrm).sum(1)).max() < 1e-4
    assert ((np.cross(u, v) * nrm).sum(1) > 0.999).all()
    m.close()
