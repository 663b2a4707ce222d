"""Print the key fields of the last JSON line of a bench.py log."""
import json
import sys

line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
d = json.loads(line)
print("ms/step", round(d["ms_per_step"], 4), "value", f"{d['value']:.4g}", "path", d.get("path"))
print("kernel_ms", d.get("kernel_ms"))
r = d.get("roofline", {})
print("roofline", r.get("kernel"), "frac", round(r.get("frac", 0), 4), "achieved", round(r.get("achieved", 0), 2))
for k in ("train_iteration", "eval", "eval_hessian"):
    if d.get(k):
        print(k, {kk: v for kk, v in d[k].items() if kk in ("ms", "stencil_points_per_s", "iterations_per_s")})
