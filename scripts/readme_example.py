"""The README usage example at small sizes (runs on one GPU)."""
import sys, numpy as np
sys.path.insert(0, ".")
from harness import mlp_spec, init_params, loss_cfg, csg_surface, uniform_box
from paper_2511_08980_b200 import FDSDF
from paper_2511_08980_b200.fdsdf import Trainer
spec = mlp_spec([3, 256, 256, 256, 256, 1], "sine")
params = init_params(spec, "siren", 0)
x = np.concatenate([csg_surface(500, 3, 1), uniform_box(500, 1.1, 2)]).astype(np.float32)
n_surface = 500
surface_pool = csg_surface(750, 3, 5).astype(np.float32)
m = FDSDF(spec, device=0, max_centers=1000)
out = m.eval(params, x, n_surface, h=5e-3, frame_seed=1)
H = m.eval_hessian(params, x, h=5e-3)
ls = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=0, lambda_eik=50, lambda_fd=1)
grad, loss = m.step(params, x, n_surface, 5e-3, ls, frame_seed=1)
tr = Trainer(m, params, surface_pool, n_pick=500, n_uniform=500, box_half=1.1, h=5e-3, loss_cfg=ls, seed=0)
for it in range(10):
    tr.iterate()
ckpt = tr.state_dict()
print("README-OK", out["K"].shape, H.shape, float(loss[4]), ckpt["t"])
