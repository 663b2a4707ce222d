"""GPU (CUDA, sm_100a) vs fp64 oracle parity, through the C ABI (libfdsdf.so).

Inputs: the seeded BASELINE.json configs (harness.make_config), at sizes the oracle finishes
in seconds but that span several tiles and a ragged tail.  Frames: the primary per-entry gate
uses the GPU's exported frames in the oracle (GIVEN mode, SURVEY §8c "two frame modes");
the self-framed mode is checked separately.  Tolerances: tests/gpu_util.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config, plane_mlp, loss_cfg, num_params  # noqa: E402
from gpu_util import ref_step, ref_eval  # noqa: E402
from gpu_util import (compare_eval, gpu_eval, per_tensor_grad_errors, LOSS_RTOL,  # noqa: E402
                      GRAD_RTOL)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


@pytest.fixture(params=["ffma", "tensor"])
def path(request):
    return request.param


def _model(spec, n, eval_only=False, path=None):
    from paper_2511_08980_b200 import FDSDF
    if path == "tensor" and (spec.get("skip_at", -1) >= 0 or max(spec["widths"][1:-1]) > 256):
        # the full tensor path needs widths <= 256 and no skip layer; such networks (C3) take the
        # default hybrid path (tensor-core forward with the skip input and weight gradient, FFMA
        # backward)
        m = FDSDF(spec, 0, max_centers=n, eval_only=eval_only)
        assert m.path == "hybrid", m.path
        return m
    m = FDSDF(spec, 0, max_centers=n, eval_only=eval_only, path=path)
    assert path is None or m.path == path
    return m


# (name, n_surface, n_uniform, h): several tiles + a ragged tail
EVAL_CASES = [("c1", 1024, 1024, None), ("c1", 37, 29, None), ("c2", 300, 213, 1e-2),
              ("c2", 256, 256, None), ("c3", 70, 61, None), ("c4", 100, 157, 1e-2)]


@pytest.mark.parametrize("name,ns,nu,h", EVAL_CASES)
def test_eval_parity_given_frames(name, ns, nu, h, path):
    c = make_config(name, ns, nu, h=h)
    m = _model(c["spec"], len(c["x"]), eval_only=True, path=path)
    g = gpu_eval(m, c)
    o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"],
                    frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    err = compare_eval(g, o)
    print(name, ns, nu, {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    assert err["mask"] == 0


@pytest.mark.parametrize("name,ns,nu,h", [("c1", 1024, 1024, 1e-2), ("c2", 200, 200, 1e-2), ("c2", 200, 200, None)])
def test_eval_parity_self_framed(name, ns, nu, h, path):
    """End-to-end: the GPU draws its own frame from its fp32 gradient; the oracle from its
    fp64 gradient with the same counter-based SplitMix64 angle (h = None: the config's own h,
    5e-3 for C2).  Every output, D and K included."""
    c = make_config(name, ns, nu, h=h)
    m = _model(c["spec"], len(c["x"]), eval_only=True, path=path)
    g = gpu_eval(m, c)
    o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], frame_seed=c["frame_seed"])
    fr = np.concatenate([o["u"], o["v"]], 1)
    assert np.max(np.abs(g["frames"] - fr)) < 1e-3
    err = compare_eval(g, o)
    print(name, h, {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    assert err["mask"] == 0


STEP_CASES = [
    ("c1", 1024, 1024, loss_cfg("ncr", "paper", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1)),  # C1a
    ("c1", 1024, 1024, loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)),  # C1b
    ("c1", 1024, 1024, loss_cfg("nsh", "paper", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1)),  # C1c
    ("c1", 1024, 1024, loss_cfg("ncr", "one", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1,
                                fd_form="square")),  # C1d
    ("c1", 53, 40, loss_cfg("ncr", "grad", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)),
    ("c2", 256, 256, None),
    ("c3", 64, 64, None),
    ("c4", 128, 128, None),
]


@pytest.mark.parametrize("case", range(len(STEP_CASES)))
def test_step_parity(case, path):
    name, ns, nu, ls = STEP_CASES[case]
    c = make_config(name, ns, nu)
    if ls is not None:
        c["loss"] = ls
    n = len(c["x"])
    m = _model(c["spec"], n, path=path)
    ev = gpu_eval(m, c, denom=c["loss"]["denom"])
    grad, loss = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"],
                    frames=(ev["frames"][:, :3], ev["frames"][:, 3:]))
    lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(c["spec"], grad, o["grad"])
    print(name, ns, nu, "loss", loss[:6], "ref", o["loss"][:6], "lerr", lerr, "gerr", gerr)
    for i in range(5):
        if o["loss"][i] != 0:
            assert lerr[i] <= LOSS_RTOL, (i, lerr)
        else:
            assert abs(loss[i]) <= 1e-12
    assert loss[5] == o["loss"][5]
    assert np.all(gerr <= GRAD_RTOL), gerr


def test_step_deterministic_and_accumulate(path):
    c = make_config("c2", 300, 300)
    m = _model(c["spec"], 600, path=path)
    g1, l1 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=7)
    g1, l1 = g1.clone(), l1.clone()
    g2, l2 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=7)
    assert torch.equal(g1, g2) and torch.equal(l1, l2)
    g3, _ = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=7, grad=g2.clone(),
                   accumulate=True)
    assert torch.allclose(g3, 2 * g1, rtol=1e-6, atol=0)
    assert m.launch_count() >= 4


def test_shard_sum_equals_full_step(path):
    """Data-parallel identity on one GPU: steps on two shards with global counts and global
    index offsets sum (grad and loss) to the full step."""
    c = make_config("c1", 512, 512)
    x, ns = c["x"], c["n_surface"]
    N = len(x)
    m = _model(c["spec"], N, path=path)
    gf, lf = m.step(c["params"], x, ns, c["h"], c["loss"], frame_seed=9)
    gf, lf = gf.cpu().numpy(), lf.cpu().numpy()
    # shard r: rows [r*N/2, (r+1)*N/2) -- shard 0 is all surface, shard 1 all uniform
    counts = (ns, N - ns, N)
    g0, l0 = m.step(c["params"], x[:512], 512, c["h"], c["loss"], counts=counts, frame_seed=9, index_offset=0)
    g0, l0 = g0.cpu().numpy(), l0.cpu().numpy()
    g1, l1 = m.step(c["params"], x[512:], 0, c["h"], c["loss"], counts=counts, frame_seed=9, index_offset=512)
    g1, l1 = g1.cpu().numpy(), l1.cpu().numpy()
    assert np.allclose(l0 + l1, lf, rtol=1e-6, atol=1e-12)
    assert np.linalg.norm(g0 + g1 - gf) <= 1e-5 * np.linalg.norm(gf)


def test_plane_mlp_zero_curvature(path):
    spec, params = plane_mlp([0.48, -0.6, 0.64], 0.1, beta=100.0, hidden_layers=3)
    x = np.random.default_rng(0).uniform(-1, 1, (300, 3)).astype(np.float32)
    m = _model(spec, 300, eval_only=True, path=path)
    o = m.eval(params, x, 150, 1e-2, frame_seed=1)
    for k in ("hess", "K", "D"):
        assert torch.max(torch.abs(o[k])).item() < 1e-3
    n = np.array([0.48, -0.6, 0.64], np.float32)
    assert np.max(np.abs(o["g"].cpu().numpy() - n)) < 1e-5


def test_errors_and_flags(path):
    from paper_2511_08980_b200 import FdsdfError
    c = make_config("c1", 16, 16)
    m = _model(c["spec"], 32, path=path)
    with pytest.raises(FdsdfError) as e:
        m.eval(c["params"], c["x"][:0], 0, 1e-2)
    assert e.value.code == "E_EMPTY"
    with pytest.raises(FdsdfError) as e:
        m.eval(c["params"], c["x"], 16, 0.0)
    assert e.value.code == "E_INVALID"
    with pytest.raises(FdsdfError) as e:
        m.eval(c["params"], np.zeros((33, 3), np.float32), 16, 1e-2)
    assert e.value.code == "E_INVALID"
    with pytest.raises(FdsdfError) as e:
        m.step(c["params"], c["x"], 0, 1e-2, c["loss"] | {"w_dm": 1.0}, counts=(0, 32, 32))
    assert e.value.code == "E_EMPTY"
    x = c["x"].copy()
    x[3, 1] = np.nan
    m.eval(c["params"], x, 16, 1e-2)
    assert m.device_flags() & 1
    assert m.device_flags() == 0  # cleared


@pytest.mark.parametrize("n", [1, 2, 33])
def test_tiny_batches(n, path):
    c = make_config("c2", max(1, n // 2), n - max(1, n // 2))
    m = _model(c["spec"], n, path=path)
    g = gpu_eval(m, c)
    o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"],
                    frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    err = compare_eval(g, o)
    assert max(err[k] for k in ("f", "g", "fuu", "fuv", "fvv")) <= 1.0, err


# ragged, unequal hidden widths (not multiples of 32 / 64): zero-padded neuron rows and K
# ranges inside the tensor tiles (MPAD 256), both activations, a 3-GEMM network; and two
# networks of the hybrid path: a skip layer whose input cat(a, x) crosses a padding boundary
# (126 + 3 -> MPAD 256) and ragged 512-padded widths with a skip layer
RAGGED = [("sine", [3, 100, 200, 150, 1], -1), ("softplus", [3, 37, 129, 90, 61, 1], -1),
          ("softplus", [3, 100, 126, 90, 1], 2), ("sine", [3, 300, 333, 290, 1], 2)]


@pytest.mark.parametrize("act,widths,skip", RAGGED)
def test_ragged_widths_eval_and_step(act, widths, skip, path):
    from harness import init_params, mlp_spec, uniform_box, csg_surface
    spec = mlp_spec(widths, act, beta=100.0, skip_at=skip)
    params = init_params(spec, "siren" if act == "sine" else "xavier", 11)
    xs = csg_surface(150, 3, 12).astype(np.float32)
    xu = uniform_box(131, 1.1, 13).astype(np.float32)
    x = np.concatenate([xs, xu])
    n, ns, h = len(x), len(xs), 1e-2
    ls = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)
    c = dict(spec=spec, params=params, x=x, n_surface=ns, h=h, frame_seed=5, loss=ls)
    m = _model(spec, n, path=path)
    g = gpu_eval(m, c)
    o = ref_eval(spec, params, x, ns, h, frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    err = compare_eval(g, o)
    print(act, widths, skip, m.path, {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    grad, loss = m.step(params, x, ns, h, ls, frame_seed=5)
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    o = ref_step(spec, params, x, ns, h, ls, frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(spec, grad, o["grad"])
    print("lerr", lerr, "gerr", gerr)
    assert np.all(lerr[o["loss"][:5] != 0] <= LOSS_RTOL), lerr
    assert np.all(gerr <= GRAD_RTOL), gerr


@pytest.mark.parametrize("om_first,om_hidden", [(30.0, 15.0), (10.0, 30.0)])
def test_sine_hidden_frequency_parity(om_first, om_hidden, path):
    """A SIREN 3->256x4->1 with omega0_first != omega0_hidden: eval
    (GIVEN frames) and step parity against the oracle -- the first / hidden frequencies are
    applied to the right layers on both paths (the closed-form pin of the oracle is
    tests/test_c_oracle_pins.py::test_sine_hidden_layer_frequency_closed_form)."""
    from harness import init_params, mlp_spec, csg_surface, uniform_box
    spec = mlp_spec([3, 256, 256, 256, 256, 1], "sine", omega0_first=om_first, omega0_hidden=om_hidden)
    params = init_params(spec, "siren", 5)
    x = np.concatenate([csg_surface(150, 3, 21), uniform_box(123, 1.1, 22)]).astype(np.float32)
    n, ns, h = len(x), 150, float(np.float32(5e-3))
    ls = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)
    c = dict(spec=spec, params=params, x=x, n_surface=ns, h=h, frame_seed=11, loss=ls)
    m = _model(spec, n, path=path)
    g = gpu_eval(m, c)
    o = ref_eval(spec, params, x, ns, h, frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    err = compare_eval(g, o)
    print(om_first, om_hidden, {k: float(v) for k, v in err.items()})
    for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K"):
        assert err[k] <= 1.0, (k, err)
    grad, loss = m.step(params, x, ns, h, ls, frame_seed=11)
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    o = ref_step(spec, params, x, ns, h, ls, frames=(g["frames"][:, :3], g["frames"][:, 3:]))
    lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(spec, grad, o["grad"])
    print("lerr", lerr, "gerr", gerr)
    assert np.all(lerr[o["loss"][:5] != 0] <= LOSS_RTOL), lerr
    assert np.all(gerr <= GRAD_RTOL), gerr


def _gap_threshold(gn, lo, hi):
    """an eps_grad in the middle of the widest gap between consecutive sorted |g| among the
    ranks [lo, hi): no centre lies near the threshold, so fp32 and fp64 take the same decision"""
    s = np.sort(gn)
    j = lo + int(np.argmax(np.diff(s[lo:hi])))
    return float(0.5 * (s[j] + s[j + 1]))


@pytest.mark.parametrize("name,ns,nu", [("c1", 300, 300), ("c2", 200, 200)])
def test_degenerate_mask_step_parity(name, ns, nu, path):
    """eps_grad near the median |g| masks about half of the centres: the GPU's
    mask, n_degenerate = loss[5], every loss term and the gradient match the oracle's; masked
    centres carry u = v = 0 and zero FD entries / D / K."""
    c = make_config(name, ns, nu)
    n = len(c["x"])
    ls = dict(loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1))
    o0 = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], frame_seed=c["frame_seed"])
    gn = np.linalg.norm(o0["g"], axis=1)
    ls["eps_grad"] = _gap_threshold(gn, int(0.4 * n), int(0.6 * n))
    m = _model(c["spec"], n, path=path)
    ev = m.eval(c["params"], c["x"], c["n_surface"], c["h"], frame_seed=c["frame_seed"], eps_grad=ls["eps_grad"])
    ev = {k: v.cpu().numpy() for k, v in ev.items()}
    mk = ev["mask"].astype(bool)
    assert np.array_equal(mk, gn >= ls["eps_grad"]) and 0.3 * n < (~mk).sum() < 0.7 * n
    assert np.all(ev["frames"][~mk] == 0) and np.all(ev["hess"][~mk] == 0)
    assert np.all(ev["K"][~mk] == 0) and np.all(ev["D"][~mk] == 0)
    grad, loss = m.step(c["params"], c["x"], c["n_surface"], c["h"], ls, frame_seed=c["frame_seed"])
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    assert m.device_flags() == 0
    o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], ls,
                    frames=(ev["frames"][:, :3], ev["frames"][:, 3:]))
    assert loss[5] == o["loss"][5] == float((~mk).sum())
    lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(c["spec"], grad, o["grad"])
    print(name, "masked", int((~mk).sum()), "lerr", lerr, "gerr", gerr)
    assert np.all(lerr <= LOSS_RTOL), lerr
    assert np.all(gerr <= GRAD_RTOL), gerr


def test_all_fd_skipped_and_nonfinite_loss_flags(path):
    """Every centre masked -> L_fd = 0, n_degenerate = N and FDSDF_FLAG_ALL_FD_SKIPPED (4);
    a non-finite output bias -> a non-finite loss and FDSDF_FLAG_NONFINITE_LOSS (2) without
    the input flag; flags are sticky until read and then cleared."""
    c = make_config("c1", 64, 64)
    n = len(c["x"])
    ls = dict(loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1), eps_grad=1e9)
    m = _model(c["spec"], n, path=path)
    grad, loss = m.step(c["params"], c["x"], c["n_surface"], c["h"], ls, frame_seed=c["frame_seed"])
    loss = loss.cpu().numpy()
    assert loss[3] == 0.0 and loss[5] == n
    o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], ls, frame_seed=c["frame_seed"])
    assert o["loss"][3] == 0.0 and o["loss"][5] == n
    assert abs(loss[4] - o["loss"][4]) <= LOSS_RTOL * abs(o["loss"][4])
    assert np.all(per_tensor_grad_errors(c["spec"], grad.cpu().numpy().astype(np.float64), o["grad"]) <= GRAD_RTOL)
    assert m.device_flags() == 4
    assert m.device_flags() == 0
    p = c["params"].copy()
    p[-1] = np.float32("nan")
    grad, loss = m.step(p, c["x"], c["n_surface"], c["h"], dict(ls, eps_grad=1e-6), frame_seed=c["frame_seed"])
    assert not np.isfinite(loss.cpu().numpy()[4])
    assert m.device_flags() == 2
    assert m.device_flags() == 0
