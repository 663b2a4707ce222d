"""fdsdf_eval_hessian: the 19-point world-axis FD Hessian on the GPU vs the
fp64 oracle (oracle.oracle_hessian, pinned in tests/test_hessian_oracle.py), through the C ABI.
Gate: the per-entry bound of the FD entries, |d| <= 1e-4 (1 + |ref|) (tests/gpu_util.py), on
seeded configs at sizes that span several tiles with ragged tails; both contraction paths;
argument errors; agreement with the tangent-frame eval on the same axis frame."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config  # noqa: E402
from oracle import oracle_hessian  # noqa: E402
from gpu_util import entry_bound  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


def _model(spec, n, path=None, eval_only=True):
    from paper_2511_08980_b200 import FDSDF
    if path == "tensor" and (spec.get("skip_at", -1) >= 0 or max(spec["widths"][1:-1]) > 256):
        m = FDSDF(spec, 0, max_centers=n, eval_only=eval_only)  # the hybrid path's tensor forward
        assert m.path == "hybrid", m.path
        return m
    return FDSDF(spec, 0, max_centers=n, eval_only=eval_only, path=path)


# (config, surface rows, uniform rows, h): C1 softplus (MPAD 128) and C2 SIREN (MPAD 256) at
# their h, plus C2 at the h = 1e-2 of the entry gate; C3 (skip layer, MPAD 512: the hybrid path
# under "tensor"); the centre counts leave ragged tiles
@pytest.mark.parametrize("name,ns,nu,h,eval_only", [("c1", 300, 211, None, True), ("c2", 333, 300, None, True),
                                                     ("c2", 200, 177, 1e-2, True), ("c2", 150, 121, None, False),
                                                     ("c3", 60, 51, None, True), ("c3", 50, 41, None, False)])
@pytest.mark.parametrize("path", ["ffma", "tensor"])
def test_hessian_parity(name, ns, nu, h, eval_only, path):
    """eval_only = False: a training context, whose centre pre-activations live in the step
    workspace (12 columns per layer) that the 2nd / 3rd passes reuse on the tensor path."""
    c = make_config(name, ns, nu, h=h)
    n = len(c["x"])
    m = _model(c["spec"], n, path=path, eval_only=eval_only)
    f = torch.empty(n, device="cuda")
    g = torch.empty(n, 3, device="cuda")
    H = m.eval_hessian(c["params"], c["x"], c["h"], f=f, g=g).cpu().numpy()
    fo, Ho = oracle_hessian(c["spec"], c["params"], c["x"], c["h"])
    err = np.abs(H - Ho) / entry_bound(Ho)
    print(name, path, "max normalised Hessian error", err.max(), "per entry", err.max(0))
    assert np.isfinite(H).all()
    assert err.max() <= 1.0
    assert np.max(np.abs(f.cpu().numpy() - fo) / entry_bound(fo)) <= 1.0
    m.close()


def test_hessian_matches_axis_frame_eval():
    """Pass 1 of the Hessian mode IS the tangent-frame eval with the GIVEN frame (e_x, e_y):
    H_xx, H_xy, H_yy equal that eval's (f_uu, f_uv, f_vv) bit for bit, and f, g equal its
    f, g."""
    c = make_config("c2", 150, 100)
    n = len(c["x"])
    m = _model(c["spec"], n)
    f = torch.empty(n, device="cuda")
    g = torch.empty(n, 3, device="cuda")
    H = m.eval_hessian(c["params"], c["x"], c["h"], f=f, g=g).cpu().numpy()
    fr = np.tile(np.array([1, 0, 0, 0, 1, 0], np.float32), (n, 1))
    o = m.eval(c["params"], c["x"], c["n_surface"], c["h"], frames=fr, eps_grad=0.0)
    hs = o["hess"].cpu().numpy()
    assert np.array_equal(H[:, 0], hs[:, 0]) and np.array_equal(H[:, 1], hs[:, 1])
    assert np.array_equal(H[:, 3], hs[:, 2])
    assert np.array_equal(f.cpu().numpy(), o["f"].cpu().numpy())
    assert np.array_equal(g.cpu().numpy(), o["g"].cpu().numpy())
    m.close()


def test_hessian_errors_and_limits():
    from paper_2511_08980_b200 import FdsdfError
    c = make_config("c1", 40, 40)
    n = len(c["x"])
    m = _model(c["spec"], n)
    ok = m.eval_hessian(c["params"], c["x"], c["h"])
    assert ok.shape == (n, 6)
    for bad_h in (0.0, -1e-2, float("nan"), float("inf")):
        with pytest.raises(FdsdfError):
            m.eval_hessian(c["params"], c["x"], bad_h)
    with pytest.raises(FdsdfError):  # n > max_centers
        m.eval_hessian(c["params"], np.concatenate([c["x"], c["x"][:1]]), c["h"])
    with pytest.raises(FdsdfError) as e:  # empty
        m.eval_hessian(c["params"], np.zeros((0, 3), np.float32), c["h"])
    assert e.value.status == 2  # FDSDF_E_EMPTY
    # a single centre (one ragged tile) and the full capacity agree with the batched call
    one = m.eval_hessian(c["params"], c["x"][5:6], c["h"]).cpu().numpy()
    assert np.allclose(one[0], ok.cpu().numpy()[5], rtol=0, atol=1e-6)
    m.close()
