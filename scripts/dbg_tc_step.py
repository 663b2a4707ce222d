"""Debug: step gradients of the tensor path vs the FFMA path on C1 / C2 subsets."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from harness import make_config
from paper_2511_08980_b200 import FDSDF

for name, ns, nu in (("c2", 256, 256), ("c1", 256, 256)):
    c = make_config(name, ns, nu)
    out = {}
    for path in ("ffma", "tensor"):
        m = FDSDF(c["spec"], 0, max_centers=len(c["x"]), path=path)
        g, l = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
        torch.cuda.synchronize()
        out[path] = (g.cpu().numpy(), l.cpu().numpy())
        m.close()
    gf, gt = out["ffma"][0], out["tensor"][0]
    print(name, "loss", out["ffma"][1][:5], out["tensor"][1][:5])
    print(name, "grad rel", np.linalg.norm(gt - gf) / np.linalg.norm(gf), "nan", np.isnan(gt).sum(),
          "max", np.abs(gt).max(), np.abs(gf).max())
    bad = np.where(~np.isfinite(gt) | (np.abs(gt - gf) > 1e-2 * np.abs(gf).max()))[0]
    print(name, "bad idx", bad[:20], len(bad))
