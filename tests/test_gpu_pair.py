"""The CTA-pair (tcgen05 cta_group::2) forward kernels (fwd_tc2.cu, opt-in via FDSDF_PAIR=1):
the same oracle gates as the default path, in a subprocess so the environment switch applies
to a fresh context."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
from harness import make_config
from gpu_util import ref_step, ref_eval
from gpu_util import compare_eval, gpu_eval, per_tensor_grad_errors
from paper_2511_08980_b200 import FDSDF
c = make_config("c2", 700, 613)
n = len(c["x"])
m = FDSDF(c["spec"], 0, max_centers=n)
ev = gpu_eval(m, c, denom=c["loss"]["denom"])
o = ref_eval(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], frames=(ev["frames"][:, :3], ev["frames"][:, 3:]),
                denom=c["loss"]["denom"], denom_pow=c["loss"]["denom_pow"])
err = compare_eval(ev, o)
assert all(err[k] <= 1.0 for k in ("f", "g", "fuu", "fuv", "fvv", "D", "K")), err
g, l = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
o = ref_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frames=(ev["frames"][:, :3], ev["frames"][:, 3:]))
l = l.cpu().numpy(); ge = per_tensor_grad_errors(c["spec"], g.cpu().numpy().astype(np.float64), o["grad"])
le = np.abs(l[:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
assert np.all(le[o["loss"][:5] != 0] <= 1e-4), le
assert np.all(ge <= 1e-3), ge
print("PAIR-OK", {k: round(float(v), 3) for k, v in err.items()}, le.max(), ge.max())
""" % (ROOT, os.path.join(ROOT, "tests"))


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


# the full grid (74 clusters, 1-2 pair tiles each), and 2 clusters (tens of tiles per cluster:
# every slot / parity / staging-block hand-off sequence runs many times, ragged last tile)
@pytest.mark.parametrize("max_sm", [None, "4"])
def test_pair_kernels_parity(max_sm):
    env = dict(os.environ, FDSDF_PAIR="1")
    if max_sm:
        env["FDSDF_MAX_SM"] = max_sm
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "PAIR-OK" in r.stdout
