"""Per-source-line (and per-file) warp-instruction and stall-sample breakdown of one kernel in an
ncu report (captured with --import-source on and -lineinfo builds).

  python scripts/ncu_regions.py REP KERNEL_REGEX [--top N] [--by-file]

Inlined helpers are attributed to their own files (act.cuh, common.cuh, tc.cuh, ...), so
--by-file separates the pair maps / sin-cos / splits from the kernel body."""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--by-file", action="store_true")
ap.add_argument("--launch-skip", type=int, default=0)
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + args.kernel, "--launch-skip", str(args.launch_skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = hdr = None
ins, stl, txt = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[0]:
        try:
            s = float(r[4] or 0)
            v = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        k = f if args.by_file else (f, int(r[0]))
        ins[k] += v
        stl[k] += s
        if not args.by_file:
            txt[k] = r[1].strip()
ti, ts = sum(ins.values()) or 1, sum(stl.values()) or 1
print(f"total warp instructions {ti:.4g}")
for k, v in ins.most_common(args.top):
    label = k if args.by_file else f"{k[0]}:{k[1]} {txt[k][:90]}"
    print(f"{100 * v / ti:5.1f}% inst {100 * stl[k] / ts:5.1f}% stall  {label}")
