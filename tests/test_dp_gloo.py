"""Data-parallel host logic on CPU (gloo, world_size 2): every rank runs the fp64 oracle on
its own shard with GLOBAL loss denominators and GLOBAL frame indices (index_offset =
rank * N_loc), the ranks SUM gradient and loss with all_reduce (the collective fdsdf_step's
FDSDF_STEP_ALLREDUCE performs with NCCL on the GPU), and the result must equal the oracle on
the union of the shards (plain SUM is exact because every term is pre-divided by
its global count)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from harness import make_config, loss_cfg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(rank, ns, nu):
    """Rank-seeded shard: ns surface rows then nu uniform rows (the prefix convention)."""
    c = make_config("c1", ns, nu)
    rng = np.random.default_rng(100 + rank)
    x = c["x"].copy()
    x[:ns] = x[rng.permutation(ns)]
    x[ns:] = np.clip(x[ns:] + rng.normal(0, 0.05, (nu, 3)).astype(np.float32), -1, 1)
    return c, x


def _worker(rank, world, port, ns, nu, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle_step
    c, x = _shard(rank, ns, nu)
    ls = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)
    counts = (ns * world, nu * world, (ns + nu) * world)
    o = oracle_step(c["spec"], c["params"], x, ns, c["h"], ls, frame_seed=c["frame_seed"],
                    index_offset=rank * (ns + nu), counts=counts)
    g = torch.tensor(o["grad"])
    l = torch.tensor(o["loss"])
    dist.all_reduce(g)
    dist.all_reduce(l)
    if rank == 0:
        out.put((g.numpy(), l.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_oracle_step_equals_union(world):
    ns, nu = 24, 20
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ns, nu, q)) for r in range(world)]
    for p in procs:
        p.start()
    g, l = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import oracle_step
    xs, surf = [], []
    for r in range(world):
        c, x = _shard(r, ns, nu)
        xs.append(x)
        surf.append(np.arange(ns + nu) < ns)
    X = np.concatenate(xs)
    ls = loss_cfg("ncr", "paper", w_dm=1, lambda_dnm=100, lambda_eik=50, lambda_fd=1)
    o = oracle_step(c["spec"], c["params"], X, None, c["h"], ls, frame_seed=c["frame_seed"],
                    surface_mask=np.concatenate(surf))
    assert np.allclose(l[:6], o["loss"][:6], rtol=1e-12, atol=1e-14)
    assert np.linalg.norm(g - o["grad"]) <= 1e-12 * np.linalg.norm(o["grad"])


def test_bench_workload_sharding_contract():
    """bench.py's per-rank workload: disjoint rank-seeded shards, global counts and global
    index offsets (host logic of the N > 1 path)."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import harness.gen as gen
    small = dict(gen.__dict__)
    try:
        gen_make = gen.make_config
        gen.make_config = lambda name, rank=0, **kw: gen_make(name, 40, 30, rank=rank)
        import harness
        harness.make_config = gen.make_config
        w0 = bench.workload("c2", 0, 4)
        w3 = bench.workload("c2", 3, 4)
    finally:
        gen.make_config = small["make_config"]
        harness.make_config = small["make_config"]
    assert w0["index_offset"] == 0 and w3["index_offset"] == 3 * 70
    assert w0["counts"] == (160, 120, 280) == w3["counts"]
    assert not np.array_equal(w0["x"], w3["x"])
    assert w0["config_json"]["parallelism"] == "dp4"
