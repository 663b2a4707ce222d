"""Diagnostic: the bench's reconstruction extra under a few loss-weight / learning-rate settings
(CSG stand-in, C2 network and batch), CD / F1 / NC after N iterations.
usage: python scripts/recon_sweep.py [iters]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from harness import make_config, csg_surface, csg_surface_normals  # noqa: E402
from paper_2511_08980_b200 import FDSDF  # noqa: E402
from paper_2511_08980_b200.fdsdf import Trainer, fdsdf_mesh_metrics  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
cfg = make_config("c2")
ns = cfg["n_surface"]
pool = csg_surface(int(ns * 1.5), 3, 100).astype(np.float32)
G, Gn = csg_surface_normals(30_000, 3, 77)
G, Gn = torch.from_numpy(G).cuda(), torch.from_numpy(Gn).cuda()
SETS = [(3000, 100, 50, 0, 5e-5, "one"), (3000, 100, 50, 3, 5e-5, "one"), (3000, 100, 50, 10, 5e-5, "one"),
        (3000, 100, 50, 30, 5e-5, "one"), (3000, 100, 50, 10, 5e-5, "paper")]
for w_dm, lam_dnm, lam_eik, lam_fd, lr, denom in SETS:
    model = FDSDF(cfg["spec"], 0, max_centers=len(cfg["x"]))
    lc = dict(cfg["loss"], w_dm=float(w_dm), lambda_dnm=float(lam_dnm), lambda_eik=float(lam_eik),
              lambda_fd=float(lam_fd), denom=denom)
    tr = Trainer(model, cfg["params"], pool, ns, len(cfg["x"]) - ns, 1.1, cfg["h"], lc, seed=4, lr=lr)
    t0 = time.perf_counter()
    for _ in range(iters):
        tr.iterate()
    torch.cuda.synchronize()
    tris, _ = model.extract_mesh(tr.params, 128)
    mm = fdsdf_mesh_metrics(tris, G, Gn, nsample=100_000, seed=1, tau=0.005)
    print(f"denom {denom} w_dm {w_dm} dnm {lam_dnm} eik {lam_eik} fd {lam_fd} lr {lr}: CDx1e3 {mm['cd'] * 1e3:.3f} "
          f"F1x1e2 {mm['f1'] * 1e2:.2f} NCx1e2 {mm['nc'] * 1e2:.2f} tris {tris.shape[0]} "
          f"({time.perf_counter() - t0:.1f} s)", flush=True)
    model.close()
