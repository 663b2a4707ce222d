"""Diagnostic: layer-0 gradient, one tile of 8 centres vs the sum of 8 single-centre steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from harness import make_config, loss_cfg, layer_shapes  # noqa: E402
from oracle import oracle_step  # noqa: E402
from gpu_util import per_tensor_grad_errors  # noqa: E402
from paper_2511_08980_b200 import FDSDF  # noqa: E402

for name, ns, nu in (("c4", 128, 128), ("c1", 64, 64)):
    c = make_config(name, ns, nu)
    n = len(c["x"])
    m = FDSDF(c["spec"], 0, max_centers=n)
    ls = loss_cfg("ncr", "one", w_dm=1, lambda_dnm=0, lambda_eik=0, lambda_fd=0)
    ev = m.eval(c["params"], c["x"], c["n_surface"], c["h"], frame_seed=c["frame_seed"])
    fr = ev["frames"].cpu().numpy()
    counts = (c["n_surface"], n - c["n_surface"], n)
    for lo, hi in ((0, 8), (0, 16), (8, 16), (0, 64), (0, n)):
        xs = c["x"][lo:hi]
        nsur = max(0, min(hi, c["n_surface"]) - lo)
        g, _ = m.step(c["params"], xs, nsur, c["h"], ls, counts=counts, frame_seed=c["frame_seed"], index_offset=lo)
        g = g.cpu().numpy().astype(np.float64)
        o = oracle_step(c["spec"], c["params"], xs, nsur, c["h"], ls, counts=counts,
                        frames=(fr[lo:hi, :3], fr[lo:hi, 3:]))
        e = per_tensor_grad_errors(c["spec"], g, o["grad"])
        print(name, lo, hi, "gerr", np.array2string(e, precision=2))
        if hi - lo == 8:
            gs = np.zeros_like(g)
            for i in range(lo, hi):
                gi, _ = m.step(c["params"], c["x"][i:i + 1], 1 if i < c["n_surface"] else 0, c["h"], ls,
                               counts=counts, frame_seed=c["frame_seed"], index_offset=i)
                gs += gi.cpu().numpy()
            e2 = per_tensor_grad_errors(c["spec"], gs, o["grad"])
            print("   sum of singles gerr", np.array2string(e2, precision=2))
            (o0, i0) = layer_shapes(c["spec"])[0]
            print("   W0 tile", g[:6], "\n   W0 sing", gs[:6], "\n   W0 ref ", o["grad"][:6])
