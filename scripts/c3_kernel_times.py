"""C3 (512-wide, skip layer) full-size step: per-kernel device times (default = hybrid path;
`python scripts/c3_kernel_times.py ffma` for the FFMA path)."""
import sys
import torch
sys.path.insert(0, ".")
from harness import make_config
from paper_2511_08980_b200 import FDSDF

c = make_config("c3")
m = FDSDF(c["spec"], 0, max_centers=len(c["x"]), path=sys.argv[1] if len(sys.argv) > 1 else None)
args = (c["params"], c["x"], c["n_surface"], c["h"], c["loss"])
m.step(*args, frame_seed=1)
torch.cuda.synchronize()
m.set_kernel_timing(True)
m.kernel_times(reset=True)
for i in range(3):
    m.step(*args, frame_seed=2 + i)
torch.cuda.synchronize()
t = m.kernel_times(reset=True)
print({k: round(v[0] / max(v[1], 1), 2) for k, v in t.items() if v[1]}, "path", m.path)
