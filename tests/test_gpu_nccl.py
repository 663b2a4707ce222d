"""The NCCL plumbing of the data-parallel step on one B200: libnccl is loaded at run
time, a world-size-1 communicator is built from fdsdf_comm_unique_id, and fdsdf_step with
FDSDF_STEP_ALLREDUCE (the in-stream ncclAllReduce of grad fp32 [P] + loss fp64 [8]) must equal
the step without it (a SUM over one rank is the identity).  The world-size-2 reduction itself is
covered on CPU by tests/test_dp_gloo.py and on one GPU by the shard-sum identity
(tests/test_gpu_parity.py::test_shard_sum_equals_full_step)."""
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


def test_allreduce_world1_is_identity_and_fdsdf_allreduce():
    from paper_2511_08980_b200 import FDSDF, FdsdfError
    from paper_2511_08980_b200 import fdsdf as F
    c = make_config("c2", 300, 300)
    m = FDSDF(c["spec"], 0, max_centers=600)
    with pytest.raises(FdsdfError) as e:  # ALLREDUCE before comm_init
        m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3, allreduce=True)
    assert e.value.code == "E_UNSUPPORTED"
    uid = F.fdsdf_comm_unique_id()
    assert len(uid) == 128
    m.comm_init(uid, 0, 1)
    g1, l1 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3)
    g1, l1 = g1.clone(), l1.clone()
    g2, l2 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3, allreduce=True)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(l1, l2)
    buf = torch.arange(1000, dtype=torch.float32, device="cuda")
    F.fdsdf_allreduce(m.ctx, buf)
    torch.cuda.synchronize()
    assert torch.equal(buf, torch.arange(1000, dtype=torch.float32, device="cuda"))
    m.close()


def test_accumulate_with_allreduce_reduces_only_this_call():
    """FDSDF_STEP_ACCUMULATE | FDSDF_STEP_ALLREDUCE: the call's own gradient is reduced in a
    context buffer and then added (d_grad += sum_r g_r), so a running sum is never multiplied by
    the world size.  At world size 1: prev + g exactly, and the loss is this call's."""
    from paper_2511_08980_b200 import FDSDF
    from paper_2511_08980_b200 import fdsdf as F
    c = make_config("c2", 200, 200)
    m = FDSDF(c["spec"], 0, max_centers=400)
    m.comm_init(F.fdsdf_comm_unique_id(), 0, 1)
    g1, l1 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3)
    g1, l1 = g1.clone(), l1.clone()
    prev = torch.linspace(-1, 1, m.P, device="cuda", dtype=torch.float32)
    g2, l2 = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3, grad=prev.clone(),
                    accumulate=True, allreduce=True)
    torch.cuda.synchronize()
    assert torch.equal(g2, prev + g1) and torch.equal(l2, l1)
    m.close()
