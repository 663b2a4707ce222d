"""Debug: SM clock, power draw and throttle reasons (nvidia-smi, 20 ms sampling) while the C2 step
runs back to back for a few seconds, with and without the bench's L2 flush between steps.
usage (under gpurun): python scripts/power_probe.py [seconds] [wgrad3]   (wgrad3: the opt-in 3-product weight gradient)"""
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from harness import make_config  # noqa: E402
from paper_2511_08980_b200 import FDSDF  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
c = make_config("c2")
m = FDSDF(c["spec"], 0, max_centers=len(c["x"]), wgrad_bf16x3="wgrad3" in sys.argv[2:])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
F = "clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown"


def run(tag, with_flush):
    p = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={F}", "--format=csv,noheader,nounits", "-lms", "20"],
                         stdout=subprocess.PIPE, text=True)
    lines = []
    th = threading.Thread(target=lambda: [lines.append(x.strip()) for x in p.stdout], daemon=True)
    th.start()
    time.sleep(0.3)
    n0 = len(lines)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 0
    e0.record()
    while time.perf_counter() - t0 < secs:
        for _ in range(20):
            if with_flush:
                flush.zero_()
            m.step(c["params"], c["x"], c["n_surface"], c["h"], c["loss"], frame_seed=steps)
            steps += 1
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    n1 = len(lines)
    p.terminate()
    rows = [[x.strip() for x in ln.split(",")] for ln in lines[n0:n1]]
    clk = sorted(float(r[0]) for r in rows if len(r) >= 5)
    pw = sorted(float(r[1]) for r in rows if len(r) >= 5)
    cap = sum(1 for r in rows if len(r) >= 5 and r[2].lower().startswith("active"))
    print(f"{tag}: {steps} steps, {e0.elapsed_time(e1) / steps:.3f} ms per step (incl. flush: {with_flush}); "
          f"samples {len(clk)}; SM MHz min/median/max {clk[0]:.0f}/{clk[len(clk) // 2]:.0f}/{clk[-1]:.0f}; "
          f"power W min/median/max {pw[0]:.0f}/{pw[len(pw) // 2]:.0f}/{pw[-1]:.0f}; sw_power_cap in {cap} samples",
          flush=True)


run("warm", False)
run("steps back to back", False)
run("steps with the 256 MiB flush", True)
