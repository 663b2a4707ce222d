"""FDSDF_CREATE_WGRAD_BF16X3 (opt-in): the weight-gradient contraction with the three leading
bf16 piece products (a0 b0 + a0 b1 + a1 b0) instead of bf16x6 -- the same oracle gates as the
default step (tests/gpu_util.py: loss 1e-4, weight gradients 1e-3 relative per tensor), on
the tensor path and the hybrid path, plus the flag's validation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config, loss_cfg  # noqa: E402
from gpu_util import ref_step  # noqa: E402
from gpu_util import gpu_eval, per_tensor_grad_errors, LOSS_RTOL, GRAD_RTOL  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


CASES = [
    ("c1", 1024, 1024, loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1), "tensor"),
    ("c2", 300, 213, None, "tensor"),
    ("c3", 64, 64, None, "hybrid"),
    ("c4", 128, 128, None, "tensor"),
]


@pytest.mark.parametrize("name,ns,nu,ls,path", CASES)
def test_step_parity_wgrad_bf16x3(name, ns, nu, ls, path):
    from paper_2511_08980_b200 import FDSDF
    c = make_config(name, ns, nu)
    if ls is not None:
        c["loss"] = ls
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n, wgrad_bf16x3=True)
    assert m.path == path, m.path
    ev = gpu_eval(m, c, denom=c["loss"]["denom"])
    grad, loss = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    grad, loss = grad.cpu().numpy().astype(np.float64), loss.cpu().numpy()
    o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"],
                    frames=(ev["frames"][:, :3], ev["frames"][:, 3:]))
    lerr = np.abs(loss[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(c["spec"], grad, o["grad"])
    print(name, path, "lerr", lerr, "gerr", gerr)
    assert np.all(lerr[o["loss"][:5] != 0] <= LOSS_RTOL), lerr
    assert np.all(gerr <= GRAD_RTOL), gerr

    # the flag changes only the weight-gradient contraction: the loss is bitwise the default's,
    # the GEMM-layer gradients differ in their last bits
    m6 = FDSDF(c["spec"], 0, max_centers=n)
    g6, l6 = m6.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    assert np.array_equal(l6.cpu().numpy(), loss)
    assert not np.array_equal(g6.cpu().numpy().astype(np.float64), grad)


def test_wgrad_bf16x3_flag_validation():
    from paper_2511_08980_b200 import FDSDF, FdsdfError
    c = make_config("c1", 16, 16)
    with pytest.raises(FdsdfError) as e:
        FDSDF(c["spec"], 0, max_centers=32, path="ffma", wgrad_bf16x3=True)
    assert e.value.code == "E_INVALID"
    # widths <= 64 with a skip layer: padded width 64, FFMA-only network
    from harness import mlp_spec
    spec = mlp_spec([3, 40, 40, 1], "softplus", skip_at=1)
    with pytest.raises(FdsdfError) as e:
        FDSDF(spec, 0, max_centers=32, wgrad_bf16x3=True)
    assert e.value.code == "E_UNSUPPORTED"
