"""Diagnostic: per-variant / per-centre layer-0 gradient error vs oracle (C4 subset)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from harness import make_config, loss_cfg
from oracle import oracle_step
from gpu_util import per_tensor_grad_errors
from paper_2511_08980_b200 import FDSDF

c = make_config("c4", 128, 128)
n = len(c["x"])
m = FDSDF(c["spec"], 0, max_centers=n)
ev = m.eval(c["params"], c["x"], c["n_surface"], c["h"], frame_seed=c["frame_seed"])
fr = ev["frames"].cpu().numpy()
gn = np.linalg.norm(ev["g"].cpu().numpy(), axis=1)
K = ev["K"].cpu().numpy()
print("min gn", np.sort(gn)[:5], "max |K|", np.sort(np.abs(K))[-5:])
variants = {
 "full": c["loss"],
 "fd_one": loss_cfg("ncr", "one", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1),
 "fd_paper": loss_cfg("ncr", "paper", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1),
 "fd_grad": loss_cfg("ncr", "grad", w_dm=0, lambda_dnm=0, lambda_eik=0, lambda_fd=1),
 "eik": loss_cfg("ncr", "one", w_dm=0, lambda_dnm=0, lambda_eik=50, lambda_fd=0),
 "dm": loss_cfg("ncr", "one", w_dm=1, lambda_dnm=0, lambda_eik=0, lambda_fd=0),
}
for k, ls in variants.items():
    g, l = m.step(c["params"], c["x"], c["n_surface"], c["h"], ls, frame_seed=c["frame_seed"])
    o = oracle_step(c["spec"], c["params"], c["x"], c["n_surface"], c["h"], ls, frames=(fr[:, :3], fr[:, 3:]))
    e = per_tensor_grad_errors(c["spec"], g.cpu().numpy().astype(np.float64), o["grad"])
    print(k, "loss", l.cpu().numpy()[4], o["loss"][4], "gerr", np.array2string(e, precision=2))
# per-centre for the worst
ls = variants["fd_paper"]
order = np.argsort(-np.abs(K))[:4]
counts = (c["n_surface"], n - c["n_surface"], n)
for i in order:
    xi = c["x"][i:i+1]
    g, l = m.step(c["params"], xi, 1 if i < c["n_surface"] else 0, c["h"], ls, counts=counts, frame_seed=c["frame_seed"], index_offset=i)
    o = oracle_step(c["spec"], c["params"], xi, 1 if i < c["n_surface"] else 0, c["h"], ls, frames=(fr[i:i+1, :3], fr[i:i+1, 3:]), counts=counts)
    e = per_tensor_grad_errors(c["spec"], g.cpu().numpy().astype(np.float64), o["grad"])
    print("centre", i, "surf", i < c["n_surface"], "gn", gn[i], "K", K[i], "loss", l.cpu().numpy()[3], o["loss"][3], "gerr", np.array2string(e, precision=2))
