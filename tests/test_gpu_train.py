"""The training iteration on the GPU vs its oracle (oracle/train_oracle.py):
fdsdf_sample bit-exact, fdsdf_adam to fp32 rounding, and a 3-iteration training loop
(sample -> step -> Adam) against oracle_step + the oracle Adam."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from harness import make_config, sphere_surface  # noqa: E402
from gpu_util import ref_step  # noqa: E402
from oracle.train_oracle import adam_step, sample_batch  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


def _model(spec, n):
    from paper_2511_08980_b200 import FDSDF
    return FDSDF(spec, 0, max_centers=n)


@pytest.mark.parametrize("n_pool,n_pick,n_unif", [(3000, 2000, 2000), (30, 20, 7), (5, 0, 33), (1, 1, 0)])
def test_sample_bit_exact(n_pool, n_pick, n_unif):
    c = make_config("c1", 16, 16)
    m = _model(c["spec"], 64)
    pool = sphere_surface(n_pool, 0.5, seed=9).astype(np.float32)
    for it in (0, 1, 17):
        x = m.sample(pool, n_pick, 1.1, n_unif, seed=1234567, iteration=it).cpu().numpy()
        ref = sample_batch(pool, n_pick, 1.1, n_unif, 1234567, it)
        assert x.shape == ref.shape
        assert np.array_equal(x.view(np.uint32), ref.view(np.uint32))


def test_sample_errors():
    from paper_2511_08980_b200 import FdsdfError
    c = make_config("c1", 16, 16)
    m = _model(c["spec"], 64)
    pool = np.zeros((10, 3), np.float32)
    with pytest.raises(FdsdfError) as e:
        m.sample(pool, 11, 1.0, 0, 0, 0)
    assert e.value.code == "E_INVALID"
    with pytest.raises(FdsdfError) as e:
        m.sample(pool, 0, 1.0, 0, 0, 0)
    assert e.value.code == "E_EMPTY"
    with pytest.raises(FdsdfError) as e:
        m.sample(pool, 1, 0.0, 1, 0, 0)
    assert e.value.code == "E_INVALID"


def test_adam_matches_oracle_and_flags():
    c = make_config("c1", 16, 16)
    m = _model(c["spec"], 64)
    P = m.P
    rng = np.random.default_rng(0)
    p0 = rng.standard_normal(P).astype(np.float32)
    p = torch.from_numpy(p0.copy()).cuda()
    mom, vel = torch.zeros(P, device="cuda"), torch.zeros(P, device="cuda")
    rp, rm, rv = p0.astype(np.float64), np.zeros(P), np.zeros(P)
    for t in range(1, 4):
        g = (rng.standard_normal(P) * np.exp(rng.uniform(-5, 1, P))).astype(np.float32)
        if t == 2:
            g[7] = np.nan
        m.adam(p, torch.from_numpy(g).cuda(), mom, vel, t, lr=1e-3)
        rp, rm, rv = adam_step(rp, g.astype(np.float64), rm, rv, t, lr=1e-3)
        rp = rp.astype(np.float32).astype(np.float64)  # parameters are stored in fp32
    pg = p.cpu().numpy().astype(np.float64)
    # fp32 parameter storage: the two sides may round the last step's result differently
    ulp = np.spacing(np.abs(rp).astype(np.float32)).astype(np.float64)
    # plus fp32 moments / fp32 gradient arithmetic: ~1e-6 of the accumulated update
    err = np.abs(pg - rp) / (ulp + 1e-6 * np.abs(rp - p0))
    print("adam max err (units of ulp(p) + 1e-6 |update|):", err.max())
    assert err.max() <= 2.0
    assert m.device_flags() & 8


def test_training_loop_matches_oracle():
    from paper_2511_08980_b200.fdsdf import Trainer
    c = make_config("c1", 16, 16)
    spec, params, lc = c["spec"], c["params"], dict(c["loss"])
    lc.update(w_dm=1.0, lambda_dnm=100.0, lambda_eik=50.0, lambda_fd=1.0)
    pool = sphere_surface(300, 0.5, seed=4).astype(np.float32)
    n_pick, n_unif, half, h, lr = 200, 200, 1.0, 1e-2, 1e-3
    m = _model(spec, n_pick + n_unif)
    tr = Trainer(m, params, pool, n_pick, n_unif, half, h, lc, seed=21, lr=lr)
    losses = []
    for _ in range(3):
        losses.append(tr.iterate().cpu().numpy().copy())
    p_gpu = tr.params.cpu().numpy().astype(np.float64)

    rp, rm, rv = params.astype(np.float64), np.zeros(len(params)), np.zeros(len(params))
    for it in range(3):
        x = sample_batch(pool, n_pick, half, n_unif, 21, it)
        fs = tr.frame_seed(it)
        o = ref_step(spec, rp.astype(np.float32), x, n_pick, h, lc, frame_seed=fs)
        lerr = abs(losses[it][4] - o["loss"][4]) / abs(o["loss"][4])
        print("iter", it, "loss", losses[it][4], "oracle", o["loss"][4], "rel", lerr)
        assert lerr <= 1e-3  # params drift apart by O(lr * 1e-5) after the first update
        rp, rm, rv = adam_step(rp, o["grad"], rm, rv, it + 1, lr=lr)
        rp = rp.astype(np.float32).astype(np.float64)  # the GPU keeps fp32 parameters
    d_gpu, d_ref = p_gpu - params, rp - params
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    print("param-update rel L2", rel)
    assert rel <= 1e-2


def test_checkpoint_resume_is_exact():
    """Trainer.state_dict / load_state_dict: 2 iterations, checkpoint, 2 more -- equals 4
    uninterrupted iterations bit for bit (parameters, moments, the iteration counter that keys
    the sampler and the frame seeds), also when resumed into a fresh context."""
    from paper_2511_08980_b200.fdsdf import Trainer
    c = make_config("c1", 16, 16)
    spec, params, lc = c["spec"], c["params"], dict(c["loss"])
    lc.update(w_dm=1.0, lambda_dnm=100.0, lambda_eik=50.0, lambda_fd=1.0)
    pool = sphere_surface(300, 0.5, seed=4).astype(np.float32)
    args = (pool, 150, 150, 1.0, 1e-2, lc)
    m = _model(spec, 300)
    ref = Trainer(m, params, *args, seed=7, lr=1e-3)
    for _ in range(4):
        ref.iterate()
    a = Trainer(m, params, *args, seed=7, lr=1e-3)
    for _ in range(2):
        a.iterate()
    st = a.state_dict()
    m2 = _model(spec, 300)
    b = Trainer(m2, np.zeros_like(params), *args, seed=0, lr=1e-3)
    b.load_state_dict(st)
    for _ in range(2):
        b.iterate()
    torch.cuda.synchronize()
    for k in ("params", "mom1", "mom2"):
        assert torch.equal(getattr(ref, k).cpu(), getattr(b, k).cpu()), k
    assert b.t == ref.t == 4
    with pytest.raises(ValueError):
        b.load_state_dict({**st, "params": st["params"][:-1]})
