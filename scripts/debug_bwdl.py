"""Debug: one hybrid-path step (layer-wise tensor backward) on tiny skip-layer networks."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from harness import init_params, mlp_spec, uniform_box, loss_cfg
from paper_2511_08980_b200 import FDSDF

widths = [int(w) for w in sys.argv[1].split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
spec = mlp_spec(widths, "softplus", beta=100.0, skip_at=2)
params = init_params(spec, "xavier", 11)
x = uniform_box(n, 1.0, 3).astype(np.float32)
m = FDSDF(spec, 0, max_centers=n)
print("path", m.path, flush=True)
g, l = m.step(params, x, n // 2, 1e-2, loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1),
              frame_seed=5)
torch.cuda.synchronize()
print("ok", l.cpu().numpy()[:5], flush=True)
