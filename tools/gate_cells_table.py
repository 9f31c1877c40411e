"""Prints the per-cell C5 table from tools/gate_cells.py's JSON (tools/)."""
import json
import sys

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1_gate_cells.json"))
print("profile", d["profile_b200"])
print("cpu", d["cpu_model_host_engine"])


def f(s):
    if "p50" not in s:  # a host path the reference refuses (CapacityError)
        return f"{'refused (' + s.get('error', '?')[:13] + ')':>29s}"
    return f"{s['p50'] * 1e3:9.3f}/{s['p95'] * 1e3:9.3f}/{s['p99'] * 1e3:9.3f}"


for c in d["cells"]:
    kk = c.get("k", c.get("m"))
    print(f"{c['op']:5s} n={c['n']:>11,} {'k' if 'k' in c else 'm'}={kk:>10,} {c['mode']:8s} cpu {f(c['cpu_only'])} "
          f"dev {f(c['always_on'])} gated {f(c['gated'])} -> {c['gate_choice']:6s} "
          f"p95x {c['gated_p95_over_best_fixed']:.2f} p99x {c['gated_p99_over_best_fixed']:.2f}")

if "cpu_model_host_engine_k_aware" in d:
    print("cpu k-aware", d["cpu_model_host_engine_k_aware"], "margin_s", d.get("margin_s_k_aware"))
    for c in d["cells"]:
        kk = c.get("k", c.get("m"))
        print(f"{c['op']:5s} n={c['n']:>11,} {kk:>10,} {c['mode']:8s} k-aware gated {f(c['gated_k_aware'])} -> "
              f"{c['gate_choice_k_aware']:6s} p95x {c['gated_k_aware_p95_over_best_fixed']:.2f} "
              f"p99x {c['gated_k_aware_p99_over_best_fixed']:.2f}")


def summary(tag, choice_key, prefix):
    cells = d["cells"]
    if choice_key not in cells[0]:
        return
    right = sum((c[choice_key] == "device") == (c["always_on"]["p50"] < c["cpu_only"].get("p50", float("inf")))
                for c in cells)
    le95 = sum(c[f"{prefix}p95_over_best_fixed"] <= 1.0 for c in cells)
    w5 = sum(c[f"{prefix}p95_over_best_fixed"] <= 1.05 for c in cells)
    print(f"{tag}: faster path chosen in {right}/{len(cells)} cells; P95 <= best fixed in {le95}, within 5% in {w5}")


summary("reference form", "gate_choice", "gated_")
summary("K-aware", "gate_choice_k_aware", "gated_k_aware_")
