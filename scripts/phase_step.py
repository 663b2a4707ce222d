"""Debug: one full-size C2 step with the phase-timing build (FDSDF_LIB=.../libfdsdf_phase.so)."""
import sys
import torch
sys.path.insert(0, ".")
from harness import make_config
from paper_2511_08980_b200 import FDSDF

c = make_config("c2")
m = FDSDF(c["spec"], 0, max_centers=len(c["x"]))
for it in range(2):
    if it == 1:
        print("---- timed step", flush=True)
    m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=c["frame_seed"])
    torch.cuda.synchronize()
