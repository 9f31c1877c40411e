"""Loads the reference-generated golden vectors (tests/golden/make_golden.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def cases(name: str) -> list[dict]:
    z = np.load(GOLDEN / f"{name}.npz")
    cols = sorted({k[:-4] for k in z.files if k.endswith("_off")})
    scalars = [k for k in z.files if not k.endswith("_off") and k not in cols]
    n = len(z[cols[0] + "_off"]) - 1
    out = []
    for i in range(n):
        case = {}
        for c in cols:
            off = z[c + "_off"]
            case[c] = z[c][off[i]:off[i + 1]]
        for s in scalars:
            v = z[s][i]
            case[s] = v.item() if hasattr(v, "item") else v
        out.append(case)
    return out


def gate_golden() -> dict:
    return json.loads((GOLDEN / "gate.json").read_text())


def npz(name: str):
    return np.load(GOLDEN / f"{name}.npz")
