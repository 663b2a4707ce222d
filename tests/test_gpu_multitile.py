"""Many tiles per CTA at oracle-sized inputs: FDSDF_MAX_SM caps the persistent grids so that
each CTA runs tens of tiles, exercising the cross-tile pipelining of the tensor kernels (the
next tile's layer 0 / top layer computed during the current tile's MMA phases, double-buffered
seeds and centre info, deferred per-centre epilogues) with ragged last tiles.  Same oracle
gates as the full-grid parity tests, in a subprocess so the environment applies to a fresh
context."""
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
name, ns, nu, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
c = make_config(name, ns, nu)
n = len(c["x"])
m = FDSDF(c["spec"], 0, max_centers=n)
assert m.path == path, m.path
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
print("MULTITILE-OK", {k: round(float(v), 3) for k, v in err.items()}, le.max(), ge.max())
""" % (ROOT, os.path.join(ROOT, "tests"))


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()


# (config, surface rows, off-surface rows, SMs, path): c2 (SIREN 256, MPAD 256) 1313 centres on
# 2 SMs -> 41 / 82 tiles per CTA in the forward / backward; c1 (softplus 64, MPAD 128) on 3 SMs;
# c3 (softplus 512 with the skip layer, hybrid path: N = 32 forward tiles of 4 centres) 131
# centres on 2 SMs -> 16-17 forward tiles per CTA, one weight-gradient split of four blocks
@pytest.mark.parametrize("name,ns,nu,sms,path", [("c2", 700, 613, 2, "tensor"), ("c1", 509, 400, 3, "tensor"),
                                                 ("c3", 70, 61, 2, "hybrid")])
def test_many_tiles_per_cta(name, ns, nu, sms, path):
    env = dict(os.environ, FDSDF_MAX_SM=str(sms))
    r = subprocess.run([sys.executable, "-c", SCRIPT, name, str(ns), str(nu), path], env=env,
                       capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "MULTITILE-OK" in r.stdout
