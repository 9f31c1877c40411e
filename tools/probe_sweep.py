"""Tuning sweep: time the resident join (build + probe kernels) for library
variants compiled with different -D shapes. Usage (GPU box):
    python tools/probe_sweep.py run  <lib.so> [nb np]
    python tools/probe_sweep.py build            # here: compile the variants
"""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
VDIR = ROOT / "paper_2601_19911_b200" / "variants"
VARIANTS = {
    "w2_b6": ["GOLP_WARP_ITEMS=2", "GOLP_PROBE_MINB=6"],
    "w2_b8": ["GOLP_WARP_ITEMS=2", "GOLP_PROBE_MINB=8"],
    "w4_b4": ["GOLP_WARP_ITEMS=4", "GOLP_PROBE_MINB=4"],
    "w4_b6": ["GOLP_WARP_ITEMS=4", "GOLP_PROBE_MINB=6"],
}


def build():
    from paper_2601_19911_b200.csrc import build as b

    VDIR.mkdir(exist_ok=True)
    for name, d in VARIANTS.items():
        b.build(out=VDIR / f"lib_{name}.so", defines=d)
        print("built", name)


def run(lib, nb=1_000_000, np_=10_000_000):
    os.environ["GOLP_B200_LIB"] = lib
    import numpy as np
    import torch

    from paper_2601_19911_b200 import _native, resident

    rng = np.random.Generator(np.random.PCG64(1))
    bk = rng.integers(0, 2 * nb, size=nb).astype(np.float64)
    pk = rng.integers(0, 2 * nb, size=np_).astype(np.float64)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    tbk, tpk = t(bk), t(pk)
    tbr = torch.arange(nb, dtype=torch.int32, device=dev)
    tpr = torch.arange(np_, dtype=torch.int32, device=dev)
    op, ob = resident.join(tbk, tbr, tpk, tpr)
    outp = torch.empty(op.numel(), dtype=torch.int32, device=dev)
    outb = torch.empty_like(outp)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    resident.set_profiling(True)
    pm, bm = [], []
    for i in range(25):
        flush.zero_()
        resident.join_build(tbk, tbr)
        resident.join_probe(tpk, tpr, outp, outb)
        kt = _native.kernel_times()
        if i >= 5:
            pm.append(kt["join_probe_ms"])
            bm.append(kt["join_build_ms"])
    ok = bool(torch.equal(outp, op) and torch.equal(outb, ob))
    print(json.dumps({"lib": Path(lib).name, "probe_ms": statistics.median(pm), "build_ms": statistics.median(bm),
                      "pairs": int(op.numel()), "stable": ok}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(sys.argv[2], *[int(x) for x in sys.argv[3:]])
