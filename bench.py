#!/usr/bin/env python
"""bench.py -- throughput of the FD curvature-regularised neural-SDF training step
(arXiv 2511.08980) on B200, through the C ABI of libfdsdf.so.

One "step" = one fdsdf_step over one batch: centre forward + grad f, random tangent frame,
the 9-point stencil of PAPER.md L83-91 (§3.1), K_FD / D_FD (L112, L121), Eq. (1) (L134-141),
the backward to every weight, and (N > 1) the NCCL allreduce of the weight gradient.

Workload (BASELINE.json configs[1], "C2"): SIREN 3->256x4->1 (omega0 = 30), 20k surface
points on a seeded CSG shape + 20k uniform points in [-1.1, 1.1]^3, h = 5e-3, FD Gaussian
curvature (PAPER denominators) + eikonal + Dirichlet.  N > 1: weak scaling, every rank owns a
fresh C2-sized shard (rank-seeded), global index offsets and global loss denominators, and
the step ends with the gradient allreduce.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c5]

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every key).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "FD-regularized SDF train steps/s & stencil points/s; % of pipe/HBM roofline"
UNIT = "stencil points/s"
FP32_LANES_PER_SM = 128          # FP32 FFMA lanes per SM (4 SMSPs x 32), B200_PROFILING.md
NOMINAL_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c2", "c5"), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the train-iteration and eval measurements")
    ap.add_argument("--no-eval-sweep", action="store_true",
                    help="skip C5e: fdsdf_eval throughput for 1e4 .. 1e7 centres (N = 1 only, 'eval_sweep')")
    ap.add_argument("--recon-iters", type=int, default=3000,
                    help="training iterations of the reconstruction extra (N = 1; 0 = skip)")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the C5 block (BASELINE configs[4]: 200k centres per GPU, every N)")
    ap.add_argument("--path", choices=("default", "ffma", "tensor"), default="default",
                    help="contraction path of the library (default: the library's choice)")
    return ap.parse_args()


def measured_bf16_peak():
    """Dense bf16 TFLOP/s: MEASURED_PEAKS.json (driver-written, burst figure), else the
    B200_PROFILING.md fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        v = float(json.load(open(p))["bf16_tflops"])
        return v, "measured (MEASURED_PEAKS.json, burst)"
    except (OSError, ValueError, KeyError):
        return 1590.0, "fallback (B200_PROFILING.md)"


def source_hash():
    """sha256 (16 hex) over the library's CUDA sources: tags the ncu DRAM capture with the build"""
    import hashlib
    d = os.path.join(ROOT, "paper_2511_08980_b200", "csrc")
    hs = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh")):
            hs.update(f.encode())
            hs.update(open(os.path.join(d, f), "rb").read())
    return hs.hexdigest()[:16]


def p_mm(spec):
    from harness import layer_shapes
    sh = layer_shapes(spec)
    return sum(o * i for o, i in sh), sum(o * i for o, i in sh[1:-1])


def pipe_peak(path, dev_index=0, sm_max_mhz=1965.0):
    """The contraction pipe's ceiling in TFLOP/s of fp32-accurate arithmetic:
    tensor / hybrid path = measured dense bf16 / 6 (bf16x6), FFMA path = SMs x 128 lanes x 2 x clock."""
    if path == "ffma":
        import torch
        nsm = torch.cuda.get_device_properties(dev_index).multi_processor_count
        return nsm * FP32_LANES_PER_SM * 2 * sm_max_mhz * 1e6 / 1e12, "alu"
    return measured_bf16_peak()[0] / 6.0, "tensor"


def roofline_of(alg_flops, ms, path, dev_index, clocks):
    """algorithmic TFLOP/s of a timed region against the pipe ceiling, with the
    fraction at the SM clock sampled during the region beside it"""
    sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    peak, bound = pipe_peak(path, dev_index, sm_max)
    ach = alg_flops / (ms * 1e-3) / 1e12
    out = {"bound": bound, "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak}
    if clocks is not None:
        out["clocks"] = clocks
        out["frac_at_run_clock"] = ach / (peak * clocks["sm_mhz"] / sm_max) if clocks.get("sm_mhz") else None
    return out


# ----------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampling (every 20 ms) of SM clock, board power and throttle reasons DURING the
    timed region: start() launches the sampler, mark() (called right before the region, after the
    sampler's start-up) discards what came before, stop() summarises the samples since mark()."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None
        self.first = 0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("FDSDF_BENCH_SMI_MS", "20")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def mark(self):
        self.first = len(self.lines)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, pw, smax, reasons = [], [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[self.first:]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            try:
                pw.append(float(f[3]))
            except ValueError:
                pass
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


# ----------------------------------------------------------------------------- oracle (CPU) arm


def _oracle_sample(cfg, nsub):
    """the first rows of each role in the workload's proportion (surface, then uniform)"""
    x, ns = cfg["x"], cfg["n_surface"]
    n = len(x)
    s = min(ns, max(1, round(nsub * ns / n)))
    u = min(n - ns, nsub - s)
    return np.concatenate([x[:s], x[ns:ns + u]]), s, u


def oracle_rate(cfg, budget_s=15.0):
    """cpu_baseline: the plain single-threaded fp64 C oracle (oracle/c/fdsdf_oracle.c) as it
    stands, on ONE host core, over a bounded sample of the workload (~budget_s of CPU work,
    sized by a timed probe).  Returns (stencil points/s, seconds per centre, cores, sample)."""
    from oracle.c_oracle import c_oracle_step

    def one(nsub):
        xs, s, u = _oracle_sample(cfg, nsub)
        t0 = time.perf_counter()
        c_oracle_step(cfg["spec"], cfg["params"], xs, s, cfg["h"], cfg["loss"], frame_seed=cfg["frame_seed"],
                      counts=cfg["counts"], need_grad=True, threads=1)
        return time.perf_counter() - t0, s, u

    dt, _, _ = one(16)
    nsub = int(min(len(cfg["x"]), max(16, budget_s / (dt / 16))))
    dt, s, u = one(nsub)
    return 9.0 * (s + u) / dt, dt / (s + u), 1, (f"one full oracle step (forward, FD epilogue, loss, weight "
                                                 f"gradient) over {s + u} of the workload's {len(cfg['x'])} centres "
                                                 f"({s} surface + {u} uniform rows), single-threaded C, fp64")


def run_reference(args):
    """The reference arm: the plain fp64 C oracle as it stands, on this box's host cores (rank 0
    alone; under torchrun the other ranks exit 0 at once).  The oracle itself is single-threaded;
    the harness runs it on `cores` contiguous row chunks in parallel threads and adds the chunks
    in order.  Each step is one oracle step over a sample of the workload's centres (surface and
    uniform rows in the workload's proportion), sized from a timed probe so that the whole
    --warmup + --steps run stays within ~3 minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.c_oracle import c_oracle_step
    cores = max(1, len(os.sched_getaffinity(0)))
    cfg = workload(args.config, 0, 1)
    n = len(cfg["x"])

    def one(nsub):
        xs, s, u = _oracle_sample(cfg, nsub)
        c_oracle_step(cfg["spec"], cfg["params"], xs, s, cfg["h"], cfg["loss"], frame_seed=cfg["frame_seed"],
                      counts=cfg["counts"], need_grad=True, threads=cores)
        return s, u

    probe = min(n, 8 * cores)
    t0 = time.perf_counter()
    one(probe)
    per_centre = (time.perf_counter() - t0) / probe
    nsub = int(min(n, max(probe, 150.0 / max(1, args.steps + args.warmup) / per_centre)))
    t_steps = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        s, u = one(nsub)
        if i >= args.warmup:
            t_steps.append(time.perf_counter() - t0)
    per = sum(t_steps) / len(t_steps)
    v = 9.0 * nsub / per
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "steps_per_s": 1.0 / per,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg["config_json"],
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"each step = one full step of the plain fp64 C oracle (forward, FD epilogue, "
                                   f"loss, weight gradient) over {s + u} of the workload's {n} centres ({s} surface "
                                   f"+ {u} uniform rows), as {cores} single-threaded row chunks in parallel"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- workload


def workload(name, rank, world):
    from harness import make_config, frame_seed
    c = make_config("c2" if name == "c2" else "c5", rank=rank)
    n = len(c["x"])
    ns = c["n_surface"]
    c["index_offset"] = rank * n
    c["counts"] = (ns * world, (n - ns) * world, n * world)
    c["frame_seed"] = frame_seed(4, 0)
    P_mm, P_gemm = p_mm(c["spec"])
    c["config_json"] = {
        "workload": ("C2: SIREN 3->256x4->1 (omega0=30, SIREN init), 20k CSG surface + 20k uniform "
                     "centres per GPU, h=5e-3, FD-NCR (paper denominators) + eikonal(50) + Dirichlet(1)")
        if name == "c2" else
        ("C5: SIREN 3->256x4->1, 100k CSG surface + 100k uniform centres per GPU, h=5e-3, FD-NCR + eik + DM"),
        "centres_per_gpu": n, "global_centres": n * world, "stencil_points_per_centre": 9,
        "params": int(len(c["params"])), "P_mm": P_mm, "h": c["h"],
        "parallelism": f"dp{world}", "l2": "flushed (256 MiB write) before every timed step",
    }
    return c


# ----------------------------------------------------------------------------- our arm


def _event_ms(stream, fn, steps, flush):
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        fn(i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / steps


def measure_extras(args, model, cfg, params, stream, flush, barrier, world, rank, dev):
    """(1) the full training iteration of PAPER.md §4: fdsdf_sample (20k of a
    30k CSG surface pool + 20k box points) -> fdsdf_step (+ allreduce) -> fdsdf_adam
    (lr 5e-5); (2) fdsdf_eval throughput (f, grad f, FD Hessian, D, K, frames, mask) on
    the same batch, and fdsdf_eval_hessian (world-axis 3x3 FD Hessian); (3)
    optionally the C5e eval sweep.  All CUDA-event timed on the stream."""
    import torch
    from harness import csg_surface
    from paper_2511_08980_b200 import FDSDF
    from paper_2511_08980_b200.fdsdf import Trainer
    out = {}
    n = len(cfg["x"])
    ns = cfg["n_surface"]
    pool = csg_surface(int(ns * 1.5), 3, 100 + rank).astype(np.float32)
    lc = cfg["loss"]
    tr = Trainer(model, params, pool, ns, n - ns, 1.1, cfg["h"], lc, seed=4 + 1000 * rank,
                 counts=cfg["counts"], index_offset=cfg["index_offset"], allreduce=world > 1)
    for _ in range(args.warmup):
        tr.iterate(stream)
    barrier()
    ms = _event_ms(stream, lambda i: tr.iterate(stream), args.steps, flush)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out["train_iteration"] = {
        "ms": ms, "iterations_per_s": 1e3 / ms, "stencil_points_per_s": 9.0 * n * world / (ms * 1e-3),
        "includes": "fdsdf_sample (20k of a 30k CSG pool + 20k box points, fresh per iteration) + "
                    "fdsdf_step" + (" + NCCL allreduce" if world > 1 else "") + " + fdsdf_adam (lr 5e-5)",
        "paper_context": "NCR-FD per-iteration time on H100, P:L399-403: 6.03 (caption unit ms) or 60.3 ms "
                         "(10-ms reading), BASELINE.md §1"}
    # eval throughput on this batch
    x = torch.from_numpy(cfg["x"]).to(dev)
    pdev = torch.from_numpy(cfg["params"]).to(dev)
    outs = model.eval(pdev, x, ns, cfg["h"], frame_seed=1, stream=stream)
    for i in range(args.warmup):
        model.eval(pdev, x, ns, cfg["h"], frame_seed=i, stream=stream, outputs=outs)
    ms_e = _event_ms(stream, lambda i: model.eval(pdev, x, ns, cfg["h"], frame_seed=i, stream=stream, outputs=outs),
                     args.steps, flush)
    out["eval"] = {"ms": ms_e, "centres": n, "stencil_points_per_s": 9.0 * n / (ms_e * 1e-3),
                   "outputs": "f, grad f, (f_uu, f_uv, f_vv), D, K, frames, mask"}
    # world-axis FD Hessian mode: 19-point stencil per centre, 3 GIVEN-frame passes
    Hb = model.eval_hessian(pdev, x, cfg["h"], stream=stream)
    for i in range(args.warmup):
        model.eval_hessian(pdev, x, cfg["h"], H=Hb, stream=stream)
    ms_h = _event_ms(stream, lambda i: model.eval_hessian(pdev, x, cfg["h"], H=Hb, stream=stream), args.steps, flush)
    out["eval_hessian"] = {"ms": ms_h, "centres": n, "stencil_points_per_s": 19.0 * n / (ms_h * 1e-3),
                           "outputs": "world-axis 3x3 FD Hessian (19-point stencil) as 3 axis-frame stencil passes"}
    if not args.no_eval_sweep and world == 1:
        from harness import csg_surface as cs, uniform_box
        sweep = []
        nmax = 10_000_000
        em = FDSDF(cfg["spec"], dev.index, max_centers=nmax, eval_only=True,
                   path=None if args.path == "default" else args.path)
        xs = np.concatenate([cs(nmax // 2, 3, 7), uniform_box(nmax - nmax // 2, 1.1, 8)]).astype(np.float32)
        xall = torch.from_numpy(xs).to(dev)
        for nn in (10_000, 30_000, 100_000, 300_000, 1_000_000, 3_000_000, 10_000_000):
            xi = xall[:nn]
            o = em.eval(pdev, xi, nn // 2, cfg["h"], frame_seed=0, stream=stream)
            for i in range(2):
                em.eval(pdev, xi, nn // 2, cfg["h"], frame_seed=i, stream=stream, outputs=o)
            # >= 1e6 centres (SURVEY §8d's eval target): enough repetitions to sample the SM clock
            reps = 5 if nn < 1_000_000 else (12 if nn == 1_000_000 else (4 if nn == 3_000_000 else 2))
            clk = None
            if nn >= 1_000_000:
                clk = ClockSampler(dev.index)
                clk.start()
                time.sleep(0.15)
                clk.mark()
            ms_s = _event_ms(stream, lambda i: em.eval(pdev, xi, nn // 2, cfg["h"], frame_seed=i, stream=stream,
                                                      outputs=o), reps, flush)
            P_mm_e = p_mm(cfg["spec"])[0]
            # eval: 20 P_mm algorithmic flops per centre (9 forward values + 1 reverse sweep)
            sweep.append({"centres": nn, "ms": ms_s, "stencil_points_per_s": 9.0 * nn / (ms_s * 1e-3),
                          "roofline": roofline_of(20.0 * P_mm_e * nn, ms_s, em.path, dev.index,
                                                  clk.stop() if clk else None)})
        em.close()
        out["eval_sweep"] = sweep
    return out


def measure_c5(args, spec, local, rank, world, dev, stream, flush, barrier):
    """BASELINE.json configs[4] at this N: 200k centres per GPU (100k CSG surface + 100k uniform,
    rank-seeded shards, global index offsets and counts), the full step with the in-step NCCL
    allreduce, event-timed, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2511_08980_b200 import FDSDF
    from paper_2511_08980_b200 import fdsdf as F
    from harness import frame_seed
    c = workload("c5", rank, world)
    n = len(c["x"])
    m = FDSDF(spec, local, max_centers=n, path=None if args.path == "default" else args.path)
    coll = setup_comm(m, world, rank, dev) if world > 1 else None
    lib_ar = coll is not None and coll.startswith("fdsdf")
    x = torch.from_numpy(c["x"]).to(dev)
    p = torch.from_numpy(c["params"]).to(dev)
    g = torch.zeros(m.P, device=dev, dtype=torch.float32)
    lo = torch.zeros(8, device=dev, dtype=torch.float64)
    lc = c["loss"]
    ls = F.make_loss(lc, c["counts"])

    def step(i):
        st = F.make_stencil(c["h"], c["n_surface"], frame_seed(4, i), c["index_offset"], None, lc["eps_grad"],
                            lc["denom"], lc["denom_pow"])
        F.fdsdf_step(m.ctx, p, x, n, st, ls, g, lo, F.STEP_ALLREDUCE if lib_ar else 0, stream)
        if world > 1 and not lib_ar:
            dist.all_reduce(g)
            dist.all_reduce(lo)

    for i in range(args.warmup):
        step(i)
    barrier()
    k = max(3, min(args.steps, 10))
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.2)
    clk.mark()
    ms = _event_ms(stream, lambda i: step(args.warmup + i), k, flush)
    clocks = clk.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ok = bool(np.isfinite(lo.cpu().numpy()[4]))
    P_mm, P_gemm = p_mm(spec)
    # whole-step algorithmic flops per GPU: (16 + 4 + 20) P_mm + 20 P_gemm per centre
    roof = roofline_of((40.0 * P_mm + 20.0 * P_gemm) * n, ms, m.path, local, clocks)
    m.close()
    return {"workload": c["config_json"]["workload"], "centres_per_gpu": n, "global_centres": n * world,
            "steps": k, "ms_per_step": ms, "steps_per_s": 1e3 / ms, "value": 9.0 * n * world / (ms * 1e-3),
            "unit": UNIT, "finite_loss": ok, "collective": coll, "roofline_step": roof}


def measure_recon(args, model, cfg, stream):
    """The paper's experiment in kind (§4) on the synthetic CSG shape: train the
    SIREN (Trainer: 20k of a 30k surface pool + 20k box points per iteration, Adam 5e-5) for
    --recon-iters iterations with and without the FD curvature term, then extract the zero level
    set on a 128^3 grid (fdsdf_eval_field + marching tetrahedra) and score it against 30k held-out
    ground-truth samples with normals: CD x10^3, F1 x10^2 (tau = 0.005), NC x10^2.
    Loss (DESIGN.md §2 item 22): the SIREN originals' weights ("hyperparameters follow the
    originals": Dirichlet 3e3, DNM 1e2 with alpha 1e2, eikonal 5e1), lambda_fd = 10 (inside the
    paper's stable range, Table tab:ablation_weights) and ||grad f|| -> 1 in every
    curvature denominator (the P:L131 replacement applied to all centres)."""
    import torch
    from harness import csg_surface, csg_surface_normals
    from paper_2511_08980_b200.fdsdf import Trainer, fdsdf_mesh_metrics
    dev = model.device
    ns = cfg["n_surface"]
    pool = csg_surface(int(ns * 1.5), 3, 100).astype(np.float32)
    G, Gn = csg_surface_normals(30_000, 3, 77)
    G, Gn = torch.from_numpy(G).to(dev), torch.from_numpy(Gn).to(dev)
    res = 128

    def score(params):
        t0 = time.perf_counter()
        tris, _ = model.extract_mesh(params, res, stream=stream)
        mm = fdsdf_mesh_metrics(tris, G, Gn, nsample=100_000, seed=1, tau=0.005, stream=stream)
        torch.cuda.synchronize()
        return {"cd_x1e3": mm["cd"] * 1e3, "f1_x1e2": mm["f1"] * 1e2, "nc_x1e2": mm["nc"] * 1e2,
                "hausdorff": mm["hausdorff"], "triangles": int(tris.shape[0]),
                "extract_and_score_s": time.perf_counter() - t0}

    def train(lambda_fd):
        lc = dict(cfg["loss"], w_dm=3000.0, lambda_dnm=100.0, alpha_dnm=100.0, lambda_eik=50.0,
                  lambda_fd=float(lambda_fd), denom="one")
        tr = Trainer(model, cfg["params"], pool, ns, len(cfg["x"]) - ns, 1.1, cfg["h"], lc, seed=4, lr=5e-5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.recon_iters):
            tr.iterate(stream)
        torch.cuda.synchronize()
        return tr.params, time.perf_counter() - t0

    init = score(cfg["params"])
    p_fd, dt = train(10.0)
    final = score(p_fd)
    p_base, _ = train(0.0)
    base = score(p_base)
    return {"iterations": args.recon_iters, "wall_s": dt, "ms_per_iteration_wall": dt * 1e3 / args.recon_iters,
            "grid": f"{res}^3 over [-1,1]^3",
            "loss": "w_dm 3e3, lambda_dnm 1e2 (alpha 1e2), lambda_eik 5e1, lambda_fd 10 (FD-NCR), ||grad f|| -> 1 "
                    "in the denominators, Adam 5e-5",
            "metrics_at_init": init, "metrics_after": final, "metrics_after_without_fd_term": base,
            "ground_truth": "30k held-out CSG surface samples with normals (harness.csg_surface_normals)",
            "note": "synthetic CSG stand-in for the ABC meshes (DESIGN.md §3); the paper trains to CD-based early "
                    "stopping (P:L153); the without-fd run is the same training with lambda_fd = 0"}


def setup_comm(model, world, rank, dev):
    """The library's own NCCL communicator (the in-step allreduce of FDSDF_STEP_ALLREDUCE): rank 0
    draws the unique id, torch.distributed broadcasts it.  Should loading / initialising it fail
    on a box, fall back to torch.distributed's NCCL all-reduce of the same two buffers on the
    same stream (reported in the JSON line)."""
    import torch
    import torch.distributed as dist
    from paper_2511_08980_b200 import fdsdf as F
    ok = 1
    try:
        uid = F.fdsdf_comm_unique_id() if rank == 0 else bytes(128)
    except F.FdsdfError:
        uid, ok = bytes(128), 0
    t = torch.tensor(list(uid) + [ok], dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0)
    ok = int(t[128].item())
    if ok:
        try:
            model.comm_init(bytes(t[:128].cpu().tolist()), rank, world)
        except F.FdsdfError as e:
            print(f"[bench] rank {rank}: fdsdf_comm_init failed ({e})", file=sys.stderr)
            ok = 0
    okt = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    return "fdsdf NCCL (in-step ncclAllReduce)" if okt.item() else "torch.distributed NCCL all_reduce"


def self_launch(args):
    """--gpus N > 1 started without torchrun: re-run this command as N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] --gpus {args.gpus} without torchrun: launching {args.gpus} ranks", file=sys.stderr)
    return subprocess.call(cmd)


def main():
    args = parse()
    # bitwise run-to-run reproducibility of the gradient allreduce at a fixed N
    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "Simple")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    from paper_2511_08980_b200 import FDSDF
    from paper_2511_08980_b200 import fdsdf as F

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"[bench] error: --gpus {args.gpus} but WORLD_SIZE={world}: a {world}-rank run cannot stand for "
              f"{args.gpus} GPUs", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = workload(args.config, rank, world)
    n = len(cfg["x"])
    spec = cfg["spec"]
    model = FDSDF(spec, local, max_centers=n, path=None if args.path == "default" else args.path)
    P = model.P
    collective = setup_comm(model, world, rank, dev) if world > 1 else None

    params = torch.from_numpy(cfg["params"]).to(dev)
    x = torch.from_numpy(cfg["x"]).to(dev)
    grad = torch.zeros(P, device=dev, dtype=torch.float32)
    loss = torch.zeros(8, device=dev, dtype=torch.float64)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lc = cfg["loss"]
    ls = F.make_loss(lc, cfg["counts"])
    lib_ar = collective is not None and collective.startswith("fdsdf")
    flags = F.STEP_ALLREDUCE if lib_ar else 0

    def stencil(step):
        from harness import frame_seed
        return F.make_stencil(cfg["h"], cfg["n_surface"], frame_seed(4, step), cfg["index_offset"], None,
                              lc["eps_grad"], lc["denom"], lc["denom_pow"])

    def one_step(i, xin=None):
        F.fdsdf_step(model.ctx, params, x if xin is None else xin, n, stencil(i), ls, grad, loss, flags, stream)
        if world > 1 and not lib_ar:
            dist.all_reduce(grad)
            dist.all_reduce(loss)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        one_step(i)
    barrier()
    launches_per_step = model.launch_count()

    # ------------------------------------------------------------------ timed region (device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    barrier()
    clk.mark()
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        one_step(args.warmup + i)
        ev[i][1].record(stream)
    barrier()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    per_step = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(per_step)
    k3 = max(1, args.steps // 3)  # the region's first and last third (this rank): the power limiter's drift
    drift = {"first_third_ms": sum(per_step[:k3]) / k3, "last_third_ms": sum(per_step[-k3:]) / k3}
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = 9.0 * n * world / (ms_per_step * 1e-3)
    assert np.isfinite(loss.cpu().numpy()[4]), "non-finite loss"

    # ------------------------------------------------------------------ per-kernel times: a second pass
    # of the same K steps with the library's per-launch events on (two cudaEventRecord around every
    # launch on the launching stream), kept out of the headline pass above
    model.set_kernel_timing(True)
    model.kernel_times(reset=True)
    barrier()
    for i in range(args.steps):
        flush.zero_()
        one_step(args.warmup + i)
    barrier()
    model.set_kernel_timing(False)
    ktimes = model.kernel_times(reset=True)

    # ------------------------------------------------------------------ e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(cfg["x"]).pin_memory()
        gh = torch.empty(P, dtype=torch.float32).pin_memory()
        lh = torch.empty(8, dtype=torch.float64).pin_memory()
        xd = torch.empty_like(x)

        def e2e_step(i):
            if world == 1 or lib_ar:
                # the public C-ABI call with host buffers: fdsdf_step_host copies x in and the
                # gradient + loss out on the stream (include/fdsdf.h)
                F.fdsdf_step_host(model.ctx, params, xh, n, stencil(i), ls, gh, lh, flags, stream)
            else:  # torch.distributed fallback collective: device step + torch copies
                xd.copy_(xh, non_blocking=True)
                one_step(i, xd)
                gh.copy_(grad, non_blocking=True)
                lh.copy_(loss, non_blocking=True)

        for i in range(2):
            e2e_step(i)
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            e2e_step(args.warmup + i)
            ev2[i][1].record(stream)
        barrier()
        e_ms = sum(a.elapsed_time(b) for a, b in ev2)
        # host wall clock per step: the call, its copies and the stream synchronisation that makes
        # the host-side gradient / loss readable (the L2 flush and its sync stay outside)
        w_s = 0.0
        barrier()
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step(args.warmup + i)
            torch.cuda.synchronize()
            w_s += time.perf_counter() - t0
        barrier()
        et = torch.tensor([e_ms, w_s * 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et[0].item()) / args.steps
        w_ms = float(et[1].item()) / args.steps
        e2e = {"value": 9.0 * n * world / (w_ms * 1e-3), "unit": UNIT, "ms_per_step": w_ms,
               "timing": "host wall clock per step (call + copies + stream sync), max over ranks",
               "device_ms_per_step": e_ms,
               "h2d_bytes_per_step": int(xh.numel() * 4), "d2h_bytes_per_step": int(P * 4 + 8 * 8),
               "call": "fdsdf_step_host (pinned host points in, gradient + loss out)" if (world == 1 or lib_ar)
               else "torch copies + fdsdf_step"}

    # ------------------------------------------------------------------ full training iteration + eval
    extras = {}
    if not args.no_extras and (world == 1 or lib_ar):
        extras = measure_extras(args, model, cfg, params, stream, flush, barrier, world, rank, dev)
    if not args.no_extras and world == 1 and model.path != "ffma":
        # the same step with the opt-in 3-product weight gradient (FDSDF_CREATE_WGRAD_BF16X3,
        # DESIGN.md §4b): reported beside the headline, never as it
        m3 = FDSDF(spec, local, max_centers=n, path=None if args.path == "default" else args.path,
                   wgrad_bf16x3=True)

        def step3(i):
            F.fdsdf_step(m3.ctx, params, x, n, stencil(i), ls, grad, loss, 0, stream)

        for i in range(args.warmup):
            step3(i)
        ms3 = _event_ms(stream, step3, args.steps, flush)
        m3.set_kernel_timing(True)
        m3.kernel_times(reset=True)
        for i in range(3):
            step3(i)
        torch.cuda.synchronize()
        kt3 = m3.kernel_times(reset=True)
        m3.close()
        extras["step_wgrad_bf16x3"] = {
            "ms_per_step": ms3, "value": 9.0 * n / (ms3 * 1e-3), "unit": UNIT,
            "wgrad_ms": kt3["wgrad"][0] / max(kt3["wgrad"][1], 1),
            "what": "opt-in FDSDF_CREATE_WGRAD_BF16X3: weight gradient with 3 bf16 piece products "
                    "(~3*2^-16 per product); forward / delta propagation bf16x6; same oracle gates"}

    # ------------------------------------------------------------------ reconstruction (NEXT-4)
    if not args.no_extras and world == 1 and args.recon_iters > 0:
        extras["reconstruction"] = measure_recon(args, model, cfg, stream)

    # ------------------------------------------------------------------ C5 (BASELINE configs[4])
    c5 = None
    if not args.no_c5 and args.config != "c5":
        c5 = measure_c5(args, spec, local, rank, world, dev, stream, flush, barrier)

    # ------------------------------------------------------------------ sustained (power-capped) figure
    # The K-step headline above lasts ~0.1 s, mostly at boost clocks; run back to back for
    # seconds the step draws the board's power limit (sw_power_cap) and the SM clock settles
    # lower.  Reported beside the headline, same step, same flush, never as the headline.
    sustained = None
    if not args.no_extras:
        ks = max(args.steps, int(2000.0 / max(ms_per_step, 1e-3)))  # ~2 s
        for i in range(ks // 4):
            flush.zero_()
            one_step(i)
        clk2 = ClockSampler(local)
        clk2.start()
        time.sleep(0.2)
        clk2.mark()
        ms_sus = _event_ms(stream, lambda i: one_step(args.warmup + i), ks, flush)
        cl2 = clk2.stop()
        ts = torch.tensor([ms_sus], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        ms_sus = float(ts.item())
        sustained = {"steps": ks, "ms_per_step": ms_sus, "value": 9.0 * n * world / (ms_sus * 1e-3), "unit": UNIT,
                     "clocks": cl2, "what": "the same step run back to back for ~2 s after ~0.5 s of the same load "
                     "(event-timed per step, flush between steps, max over ranks)"}

    # ------------------------------------------------------------------ roofline of the dominant kernel
    P_mm, P_gemm = p_mm(spec)
    path = model.path
    # algorithmic flops per launch: column-units x 2 P_mm x centres
    if path == "tensor":
        alg = {
            "fwd": 16.0 * P_mm * n,        # the 8 stencil-neighbour evaluations (pair kernel)
            "fwd_centre": 4.0 * P_mm * n,  # f(x0) + the grad-f sweep (centre kernel)
            "bwd": 20.0 * P_mm * n,        # delta through 9 evaluations + the grad-f path
            "wgrad": 20.0 * P_gemm * n,    # dW of the GEMM layers: 10 column-units
        }
    else:
        alg = {
            "fwd": 20.0 * P_mm * n,      # 9 stencil values + 1 reverse sweep for grad f
            "bwd": 20.0 * P_mm * n,      # delta through 9 evaluations + the grad-f path
            "wgrad": 20.0 * P_gemm * n,  # dW of the GEMM layers: 10 column-units
        }
    kms = {k: (v[0] / v[1] if v[1] else 0.0) for k, v in ktimes.items()}
    dom = max(alg, key=lambda k: kms[k])
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    ffma_peak = nsm * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    achieved = alg[dom] / (kms[dom] * 1e-3) / 1e12
    traffic, traffic_note = None, "no ncu capture of this build in profiles/"
    prof = os.path.join(ROOT, "profiles", "ncu_dram_per_launch.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("build") == source_hash():
                traffic = pj["per_launch"].get(dom)
                traffic_note = f"ncu --set full dram__bytes_read+write of this build ({pj.get('capture', '')})"
            else:
                traffic_note = "profiles/ncu_dram_per_launch.json is from another build of csrc/: not reported"
        except (OSError, ValueError, KeyError):
            pass
    if path == "tensor":
        # fp32-accurate contraction as 6 bf16 tensor-core products (bf16x6):
        # its ceiling is the measured dense bf16 peak / 6
        bf16, src = measured_bf16_peak()
        peak = bf16 / 6.0
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note,
                "peak_note": f"bf16x6: {src} dense bf16 {bf16:.1f} TFLOP/s / 6 bf16 MMAs per fp32-accurate MAC",
                "frac_of_fp32_ffma_peak": achieved / ffma_peak,
                "frac_at_run_clock": (achieved / (peak * clocks["sm_mhz"] / sm_max)) if clocks.get("sm_mhz") else None}
    else:
        peak = ffma_peak
        roof = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_note": f"fp32 FFMA: {nsm} SMs x {FP32_LANES_PER_SM} lanes x 2 x {sm_max:.0f} MHz (clocks.max.sm)",
                "frac_at_run_clock": (achieved / (peak * clocks["sm_mhz"] / sm_max)) if clocks.get("sm_mhz") else None}
    step_alg = sum(alg.values())
    kernel_ms = {k: round(v, 4) for k, v in kms.items() if ktimes[k][1]}
    # the same model for every contraction kernel: achieved algorithmic TFLOP/s and its fraction
    # of the roofline's peak (the dominant kernel is `roofline` above)
    roof["per_kernel"] = {k: {"achieved": alg[k] / (kms[k] * 1e-3) / 1e12,
                              "frac": alg[k] / (kms[k] * 1e-3) / 1e12 / peak}
                          for k in alg if kms.get(k)}

    # ------------------------------------------------------------------ CPU oracle baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, per_centre, cores, sample = oracle_rate(cfg)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "s_per_centre": per_centre, "s_per_full_step_extrapolated": per_centre * n}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "steps_per_s": 1e3 / ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded CSG + uniform box; DESIGN.md §3)", "config": cfg["config_json"],
            "roofline": roof, "step_alg_tflops": step_alg / (ms_per_step * 1e-3) / 1e12,
            "kernel_ms": kernel_ms, "path": path,
            "precision": ("bf16x6: fp32 operands split exactly into 3 bf16 pieces, 6 tcgen05 products, fp32 "
                          "accumulation" if path == "tensor" else "fp32 FFMA"), "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps), "clocks": clocks, **extras,
            "collective": collective, "c5": c5, "sustained": sustained, "ms_per_step_drift": drift,
            "wall_s_timed_region": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    model.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
