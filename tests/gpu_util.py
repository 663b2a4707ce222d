"""Shared helpers for the GPU parity tests: run the CUDA path through the C ABI binding and the
fp64 oracle on identical seeded inputs, and compare with the tolerances of BASELINE.json
north_star (read concretely in SURVEY.md §8c and DESIGN.md §5)."""
from __future__ import annotations

import os

import numpy as np

from harness import make_config
from oracle.c_oracle import c_oracle_step, c_oracle_eval

# The parity reference is the plain single-threaded fp64 C oracle (BASELINE.json north_star;
# oracle/c/fdsdf_oracle.c, pinned by tests/test_c_oracle_pins.py).  The harness runs it on
# contiguous row chunks in parallel threads (each call single-threaded) and adds the chunks in
# order; the oracle's arithmetic per centre is unchanged.
NTHREADS = max(1, min(32, os.cpu_count() or 1))


def ref_step(*args, **kw):
    kw.setdefault("threads", NTHREADS)
    return c_oracle_step(*args, **kw)


def ref_eval(*args, **kw):
    kw.setdefault("threads", NTHREADS)
    return c_oracle_eval(*args, **kw)

ENTRY_TOL = 1e-4     # |d| <= 1e-4 (1 + |ref|) per point value and FD Hessian entry (h = 1e-2)
LOSS_RTOL = 1e-4     # relative, each loss component and the total
GRAD_RTOL = 1e-3     # relative L2 per parameter tensor


def sub_config(name, ns=None, nu=None, h=None):
    c = make_config(name, ns, nu, h=h)
    return c


def gpu_eval(model, c, frames=None, frame_seed=None, denom="paper"):
    o = model.eval(c["params"], c["x"], c["n_surface"], c["h"],
                   frame_seed=c["frame_seed"] if frame_seed is None else frame_seed,
                   index_offset=c.get("index_offset", 0), frames=frames, denom=denom,
                   denom_pow=c["loss"].get("denom_pow", 4))
    return {k: v.cpu().numpy() for k, v in o.items()}


def entry_bound(ref):
    return ENTRY_TOL * (1.0 + np.abs(ref))


def d_bound(fuu, fuv, fvv):
    """|dD| bound propagated from the per-entry bound."""
    return ENTRY_TOL * ((1 + np.abs(fuu)) * np.abs(fvv) + (1 + np.abs(fvv)) * np.abs(fuu)
                        + 2 * (1 + np.abs(fuv)) * np.abs(fuv)) + 1e-6


def compare_eval(g, o, check_frames=True):
    """g: GPU eval dict, o: oracle dict.  Returns dict of max normalised errors (<= 1 passes)."""
    res = {}
    res["f"] = np.max(np.abs(g["f"] - o["f"]) / entry_bound(o["f"]))
    res["g"] = np.max(np.abs(g["g"] - o["g"]) / entry_bound(o["g"]))
    res["fuu"] = np.max(np.abs(g["hess"][:, 0] - o["fuu"]) / entry_bound(o["fuu"]))
    res["fuv"] = np.max(np.abs(g["hess"][:, 1] - o["fuv"]) / entry_bound(o["fuv"]))
    res["fvv"] = np.max(np.abs(g["hess"][:, 2] - o["fvv"]) / entry_bound(o["fvv"]))
    tD = d_bound(o["fuu"], o["fuv"], o["fvv"])
    res["D"] = np.max(np.abs(g["D"] - o["D"]) / tD)
    den = np.where(np.abs(o["D"]) > 0, np.abs(o["D"]) / np.maximum(np.abs(o["K"]), 1e-300), 1.0)
    den = np.where(np.abs(o["K"]) > 0, den, 1.0)
    tK = (tD + 1e-4 * np.abs(o["D"])) / den + 1e-6
    res["K"] = np.max(np.abs(g["K"] - o["K"]) / tK)
    res["mask"] = float(np.sum(g["mask"].astype(bool) != o["mask"]))
    return res


def per_tensor_grad_errors(spec, g, ref):
    from harness import layer_shapes
    out = []
    off = 0
    tot = np.linalg.norm(ref)
    for (o_, i_) in layer_shapes(spec):
        for size in (o_ * i_, o_):
            a, b = g[off:off + size], ref[off:off + size]
            nb = np.linalg.norm(b)
            if nb < 1e-9 * tot:
                out.append(np.linalg.norm(a) / (1e-6 * tot + 1e-300) * 1e-3 if tot > 0 else 0.0)
            else:
                out.append(np.linalg.norm(a - b) / nb)
            off += size
    return np.array(out)
