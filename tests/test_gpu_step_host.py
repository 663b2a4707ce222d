"""fdsdf_step_host (include/fdsdf.h): the training step with HOST buffers -- points in, gradient
and loss out, the copies enqueued by the library -- is bitwise the device-pointer step; it
accumulates with FDSDF_STEP_ACCUMULATE and validates its pointers."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


@pytest.mark.parametrize("name,ns,nu", [("c2", 300, 213), ("c3", 40, 31)])
def test_step_host_matches_device_step(name, ns, nu):
    from paper_2511_08980_b200 import FDSDF
    from paper_2511_08980_b200 import fdsdf as F
    c = make_config(name, ns, nu)
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n)
    g_dev, l_dev = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    lc = c["loss"]
    st = F.make_stencil(c["h"], c["n_surface"], c["frame_seed"], 0, None, lc["eps_grad"], lc["denom"],
                        lc["denom_pow"])
    ls = F.make_loss(lc, (c["n_surface"], n - c["n_surface"], n))
    params = torch.from_numpy(c["params"]).cuda()
    xh = torch.from_numpy(c["x"]).pin_memory()
    gh = torch.full((m.P,), np.nan, dtype=torch.float32).pin_memory()
    lh = torch.full((8,), np.nan, dtype=torch.float64).pin_memory()
    F.fdsdf_step_host(m.ctx, params, xh, n, st, ls, gh, lh)
    torch.cuda.synchronize()
    assert torch.equal(gh, g_dev.cpu()) and torch.equal(lh, l_dev.cpu())

    # ACCUMULATE: the context's gradient buffer keeps the running sum
    F.fdsdf_step_host(m.ctx, params, xh, n, st, ls, gh, lh, F.STEP_ACCUMULATE)
    torch.cuda.synchronize()
    g2, _ = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"],
                   grad=g_dev.clone(), accumulate=True)
    assert torch.equal(gh, g2.cpu())

    # pageable host memory works too (synchronous copies)
    xp, gp, lp = torch.from_numpy(c["x"].copy()), torch.empty(m.P), torch.empty(8, dtype=torch.float64)
    F.fdsdf_step_host(m.ctx, params, xp, n, st, ls, gp, lp)
    torch.cuda.synchronize()
    assert torch.equal(gp, g_dev.cpu())
    m.close()


def test_step_host_errors():
    from paper_2511_08980_b200 import FDSDF, FdsdfError
    from paper_2511_08980_b200 import fdsdf as F
    c = make_config("c1", 16, 16)
    n = len(c["x"])
    lc = c["loss"]
    st = F.make_stencil(c["h"], c["n_surface"], 0, 0, None, lc["eps_grad"], lc["denom"], lc["denom_pow"])
    ls = F.make_loss(lc, (c["n_surface"], n - c["n_surface"], n))
    params = torch.from_numpy(c["params"]).cuda()
    m = FDSDF(c["spec"], 0, max_centers=n)
    xh, gh, lh = torch.from_numpy(c["x"]), torch.empty(m.P), torch.empty(8, dtype=torch.float64)
    with pytest.raises(FdsdfError) as e:
        F.fdsdf_step_host(m.ctx, params, xh, n, st, ls, None, lh)
    assert e.value.code == "E_INVALID"
    with pytest.raises(FdsdfError) as e:
        F.fdsdf_step_host(m.ctx, params, xh, n + 1, st, ls, gh, lh)  # n > max_centers
    assert e.value.code == "E_INVALID"
    with pytest.raises(ValueError):
        F.fdsdf_step_host(m.ctx, params, xh.cuda(), n, st, ls, gh, lh)
    me = FDSDF(c["spec"], 0, max_centers=n, eval_only=True)
    with pytest.raises(FdsdfError) as e:
        F.fdsdf_step_host(me.ctx, params, xh, n, st, ls, gh, lh)
    assert e.value.code == "E_INVALID"
