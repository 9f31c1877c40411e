"""Builds library variants of the partitioned probe kernel (tools/, here):
    python tools/part_probe_variants.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200.csrc import build as b  # noqa: E402

V = Path(__file__).resolve().parents[1] / "paper_2601_19911_b200" / "variants"
V.mkdir(exist_ok=True)
for name, d in {"so_12_4": ["GOLP_SORT_ITEMS=12", "GOLP_SORT_MINB=4"],
                "so_12_3": ["GOLP_SORT_ITEMS=12", "GOLP_SORT_MINB=3"],
                "so_16_3": ["GOLP_SORT_ITEMS=16", "GOLP_SORT_MINB=3"],
                "so_8_4": ["GOLP_SORT_ITEMS=8", "GOLP_SORT_MINB=4"],
                "so_20_2": ["GOLP_SORT_ITEMS=20", "GOLP_SORT_MINB=2"]}.items():
    b.build(out=V / f"lib_{name}.so", defines=d)
    log = (V.parent / "build_ptxas.log").read_text()
    i = log.find("sort_pass_kernel")
    print(name, log[i:i + 400].split("\n")[2:4])
