"""Small eval + step on both paths (C1 padded-128 and a C2 subset) for compute-sanitizer runs."""
import sys
sys.path.insert(0, ".")
import torch
from harness import make_config
from paper_2511_08980_b200 import FDSDF

for name, ns, nu in (("c1", 40, 33), ("c2", 70, 61)):
    c = make_config(name, ns, nu)
    for path in ("tensor", "ffma"):
        m = FDSDF(c["spec"], 0, max_centers=len(c["x"]), path=path)
        m.eval(c["params"], c["x"], c["n_surface"], c["h"], frame_seed=1)
        g, l = m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=1)
        torch.cuda.synchronize()
        print(name, path, float(l[4]))
        m.close()
print("SANITIZE-DONE")
