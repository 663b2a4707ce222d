"""Summarise ncu output into profiles/ (tracked).

  python scripts/ncu_summary.py --round 1 --launches gpurun_out/launches.csv \
      --rep gpurun_out/prof_r01.ncu-rep

Writes profiles/rNN_launches.csv (the raw launch list), profiles/rNN_launch_shares.md (per kernel:
launches, total and mean device time, share of all of this library's kernel time),
profiles/rNN_ncu_full.md (key --set full metrics of the captured kernels) and
profiles/ncu_dram_per_launch.json (dram read+write bytes per launch, read by bench.py for
roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
TAG = ""
OURS = re.compile(r"(fwd_kernel|bwd_kernel|wgrad_kernel|finalize_kernel|pack_kernel|fwd_tc_kernel|bwd_tc_kernel|"
                  r"wgrad_tc_kernel|pack_tc_kernel|bwdl_tc_kernel)")
FWD_TC_MODE = re.compile(r"fwd_tc_kernel<\s*(?:\(int\))?\d+,\s*(?:\(int\))?\d+,\s*(?:\(int\))?([12])>")
# kernel -> the bench's timing slot name (bench.py kernel_ms keys)
TC_SLOT = {"bwd_tc_kernel": "bwd", "wgrad_tc_kernel": "wgrad", "pack_tc_kernel": "pack_tc", "bwdl_tc_kernel": "bwd"}

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU inst %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
]


def short(name):
    m = FWD_TC_MODE.search(name)
    if m:
        return "fwd_centre" if m.group(1) == "1" else "fwd"
    m = OURS.search(name)
    if not m:
        return name.split("(")[0][:60]
    return TC_SLOT.get(m.group(1), m.group(1).replace("_kernel", ""))


def launches(path, rnd):
    shutil.copy(path, os.path.join(PROF, f"r{rnd:02d}{TAG}_launches.csv"))
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi])
    mine = {"fwd", "fwd_centre", "bwd", "wgrad", "finalize", "pack", "pack_tc"}
    ours_tot = sum(v[1] for k, v in agg.items() if k in mine)
    out = [f"# Round {rnd} launch list summary (ncu --metrics gpu__time_duration.sum --clock-control none)",
           "", "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.", "",
           "| kernel | launches | total ms | mean ms | share of fdsdf kernel time |", "|---|---|---|---|---|"]
    for k, (n, t) in agg.items():
        ours = k in mine
        share = f"{100 * t / ours_tot:.1f}%" if ours and ours_tot else "(torch / harness)"
        out.append(f"| {k} | {n} | {t / 1e6:.3f} | {t / n / 1e6:.4f} | {share} |")
    open(os.path.join(PROF, f"r{rnd:02d}{TAG}_launch_shares.md"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(rep, rnd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    names = [short(r[idx["Kernel Name"]]) for r in data]
    out = [f"# Round {rnd} `ncu --set full` capture ({os.path.basename(rep)})", "",
           "| metric | unit | " + " | ".join(names) + " |", "|---|---|" + "---|" * len(names)]
    dram = {}
    for key, label in FULL_METRICS:
        if key not in idx:
            continue
        out.append(f"| {label} (`{key}`) | {units[idx[key]]} | " + " | ".join(r[idx[key]] for r in data) + " |")
    for r, nm in zip(data, names):
        def val(k):
            u = units[idx[k]]
            v = float(r[idx[k]])
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        dram[nm] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and
              h.endswith("_per_issue_active.ratio")]
    out += ["", "Warp stall reasons (per issue-active cycle, > 0.05 anywhere):", "",
            "| stall | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
    for h in stalls:
        vals = [float(r[idx[h]] or 0) for r in data]
        if max(vals) > 0.05:
            out.append(f"| {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} | "
                       + " | ".join(f"{v:.2f}" for v in vals) + " |")
    open(os.path.join(PROF, f"r{rnd:02d}{TAG}_ncu_full.md"), "w").write("\n".join(out) + "\n")
    import sys
    sys.path.insert(0, ROOT)
    from bench import source_hash  # the build tag bench.py checks before it reports roofline.traffic
    json.dump({"build": source_hash(), "capture": os.path.basename(rep), "per_launch": dram},
              open(os.path.join(PROF, "ncu_dram_per_launch.json"), "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", default="", help="file-name suffix, e.g. _tc")
    a = ap.parse_args()
    TAG = a.tag
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.round)
    if a.rep:
        full(a.rep, a.round)
