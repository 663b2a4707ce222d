"""Quick look at an ncu report: key metrics, top stall reasons and the hottest source lines per kernel.
usage: python scripts/ncu_quick.py REP [kernel-regex] [nlines]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 12
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size"]
for d in data:
    name = d[hdr.index("Kernel Name")]
    if kre and not re.search(kre, name):
        continue
    print("==", name[:60])
    print("   ", {w.split("__")[1][:32]: d[hdr.index(w)] for w in want if w in hdr})
    st = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    vals = sorted([(float(d[hdr.index(h)] or 0), h) for h in st], reverse=True)[:7]
    tot = sum(float(d[hdr.index(h)] or 0) for h in st) or 1
    print("    stalls:", [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), round(100 * v / tot, 1)) for v, h in vals])
if kre:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    # sections: a "Kernel Name" row, then a header row with "Source", then data rows
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            secs.append(cur)
        elif cur is not None and cur[1] is None and "Source" in r:
            cur[1] = r
        elif cur is not None and cur[1] is not None:
            cur[2].append(r)
    for name, h, data in secs:
        if not re.search(kre, name):
            continue
        iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = [r for r in data if len(r) > iW]
        tot = sum(float(r[iW] or 0) for r in data) or 1
        print("--", name[:70])
        for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:nl]:
            print(f"   {100 * float(r[iW]) / tot:5.1f}% {r[0][-5:]} {r[iS][:100]}")
