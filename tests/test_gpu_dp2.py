"""Two processes on cuda:0 run the data-parallel step of SURVEY §8e through the C ABI: each rank
steps its own shard (rank-seeded rows) with the GLOBAL loss denominators and GLOBAL frame indices
(index_offset = rank * N_loc), and the two gradients / losses are summed with a gloo all_reduce
on the host (NCCL refuses two ranks on one device; the library's in-step ncclAllReduce is the same
SUM).  The sum must equal one process stepping the union of the shards (relative 1e-5) and the
fp64 C oracle on the union (the parity gates).  Kernels of the two ranks never wait on each other."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %r); sys.path.insert(0, %r)
from harness import make_config
from paper_2511_08980_b200 import FDSDF
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
NS, NU = 300, 260
c = make_config("c2", NS, NU, rank=rank)
x = c["x"]
counts = (NS * world, NU * world, (NS + NU) * world)
m = FDSDF(c["spec"], 0, max_centers=len(x))
g, l = m.step(c["params"], x, NS, c["h"], c["loss"], counts=counts, frame_seed=c["frame_seed"],
              index_offset=rank * (NS + NU))
ev = m.eval(c["params"], x, NS, c["h"], frame_seed=c["frame_seed"], index_offset=rank * (NS + NU))
g, l, fr = g.cpu().double(), l.cpu(), ev["frames"].cpu()
dist.all_reduce(g)
dist.all_reduce(l)
xs = [torch.zeros_like(torch.from_numpy(x)) for _ in range(world)]
frs = [torch.zeros_like(fr) for _ in range(world)]
dist.all_gather(xs, torch.from_numpy(x))
dist.all_gather(frs, fr)
if rank == 0:
    np.savez(sys.argv[1], grad=g.numpy(), loss=l.numpy(), x=torch.cat(xs).numpy(), frames=torch.cat(frs).numpy())
dist.barrier()
dist.destroy_process_group()
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_sharded_step_equals_union(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_08980_b200._build import build
    build()
    script = tmp_path / "dp2.py"
    script.write_text(SCRIPT % (ROOT, os.path.join(ROOT, "tests")))
    out = tmp_path / "dp2.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script), str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = np.load(out)
    from harness import make_config
    from paper_2511_08980_b200 import FDSDF
    from gpu_util import ref_step, per_tensor_grad_errors, LOSS_RTOL, GRAD_RTOL
    NS, NU = 300, 260
    x = d["x"]
    N = len(x)
    surf = np.concatenate([np.arange(NS + NU) < NS] * 2)
    c = make_config("c2", NS, NU)
    # one process on the union: rows of rank 1 follow rank 0's (global index = row)
    perm = np.concatenate([np.where(surf)[0], np.where(~surf)[0]])
    m = FDSDF(c["spec"], 0, max_centers=N)
    # the union step needs the surface prefix convention: reorder rows, keep the global frame
    # index of each row by passing the frames the two ranks drew (GIVEN mode)
    fr = d["frames"][perm]
    g1, l1 = m.step(c["params"], x[perm], int(surf.sum()), c["h"], c["loss"], frames=fr)
    g1, l1 = g1.cpu().numpy().astype(np.float64), l1.cpu().numpy()
    assert np.allclose(d["loss"], l1, rtol=1e-5, atol=0)
    assert np.linalg.norm(d["grad"] - g1) <= 1e-5 * np.linalg.norm(g1)
    o = ref_step(c["spec"], c["params"], x, 0, c["h"], c["loss"], frames=(d["frames"][:, :3], d["frames"][:, 3:]),
                 surface_mask=surf, gidx=np.arange(N))
    lerr = np.abs(d["loss"][:5] - o["loss"][:5]) / np.maximum(np.abs(o["loss"][:5]), 1e-30)
    gerr = per_tensor_grad_errors(c["spec"], d["grad"], o["grad"])
    print("dp2 lerr", lerr, "gerr", gerr, "n_deg", d["loss"][5], o["loss"][5])
    assert np.all(lerr[o["loss"][:5] != 0] <= LOSS_RTOL) and np.all(gerr <= GRAD_RTOL)
    assert d["loss"][5] == o["loss"][5]
