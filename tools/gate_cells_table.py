"""Prints the per-cell C5 table from tools/gate_cells.py's JSON (tools/)."""
import json
import sys

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1_gate_cells.json"))
print("profile", d["profile_b200"])
print("cpu", d["cpu_model_host_engine"])


def f(s):
    return f"{s['p50'] * 1e3:9.3f}/{s['p95'] * 1e3:9.3f}/{s['p99'] * 1e3:9.3f}"


for c in d["cells"]:
    kk = c.get("k", c.get("m"))
    print(f"{c['op']:5s} n={c['n']:>11,} {'k' if 'k' in c else 'm'}={kk:>10,} {c['mode']:8s} cpu {f(c['cpu_only'])} "
          f"dev {f(c['always_on'])} gated {f(c['gated'])} -> {c['gate_choice']:6s} "
          f"p95x {c['gated_p95_over_best_fixed']:.2f} p99x {c['gated_p99_over_best_fixed']:.2f}")
