"""Builds library variants of the partitioned probe kernel (tools/, here):
    python tools/part_probe_variants.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200.csrc import build as b  # noqa: E402

V = Path(__file__).resolve().parents[1] / "paper_2601_19911_b200" / "variants"
V.mkdir(exist_ok=True)
for name, d in {"bi_256_4": [],
                "bi_512_2": ["GOLP_BUILD_THREADS=512", "GOLP_BUILD_ITEMS=2"],
                "bi_256_1": ["GOLP_BUILD_ITEMS=1"],
                "bi_512_1": ["GOLP_BUILD_THREADS=512", "GOLP_BUILD_ITEMS=1"],
                "bi_1024_2": ["GOLP_BUILD_THREADS=1024", "GOLP_BUILD_ITEMS=2"]}.items():
    b.build(out=V / f"lib_{name}.so", defines=d)
    log = (V.parent / "build_ptxas.log").read_text()
    i = log.find("join_insert_kernel")
    print(name, log[i:i + 400].split("\n")[2:4])
