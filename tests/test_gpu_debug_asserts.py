"""T6 stand-in: compute-sanitizer is refused on this GPU pool, so a bounds-checked
build of the library (-DFDSDF_DEBUG_ASSERT: device-side asserts on every computed shared-memory,
TMEM-column and global index of the tensor kernels, common.cuh FDSDF_ASSERT) runs eval, step,
the Hessian mode and a training iteration with many tiles per CTA and ragged tails, in a
subprocess; an assert traps the kernel (non-zero exit) and prints its location."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT = os.path.join(ROOT, "paper_2511_08980_b200", "variants", "libfdsdf_dbg.so")

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from harness import make_config, csg_surface
from paper_2511_08980_b200 import FDSDF
from paper_2511_08980_b200.fdsdf import Trainer
for name, ns, nu in (("c1", 301, 257), ("c2", 333, 301)):
    c = make_config(name, ns, nu)
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n)
    assert m.path == "tensor"
    ev = m.eval(c["params"], c["x"], c["n_surface"], c["h"], frame_seed=3)
    g, l = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=3)
    H = m.eval_hessian(c["params"], c["x"], c["h"])
    pool = csg_surface(int(1.5 * ns), 3, 9).astype(np.float32)
    tr = Trainer(m, c["params"], pool, ns, nu, 1.1, c["h"], c["loss"], seed=5)
    for _ in range(2):
        tr.iterate()
    torch.cuda.synchronize()
    assert np.isfinite(l.cpu().numpy()).all() and np.isfinite(H.cpu().numpy()).all()
    m.close()
print("DEBUG-ASSERT-RUN-OK")
""" % ROOT


@pytest.fixture(scope="module")
def debug_lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200 import _build
    newest = _build._newest_input()
    if not os.path.exists(VARIANT) or os.path.getmtime(VARIANT) < newest:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "build_variant.py"), "dbg",
                            "-DFDSDF_DEBUG_ASSERT"], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
    return VARIANT


def test_bounds_checked_build_runs_clean(debug_lib):
    env = dict(os.environ, FDSDF_LIB=debug_lib, FDSDF_MAX_SM="3")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert "FDSDF_ASSERT" not in out
    assert r.returncode == 0 and "DEBUG-ASSERT-RUN-OK" in r.stdout
