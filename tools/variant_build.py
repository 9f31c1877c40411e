"""Build tuning variants of libgolp_b200.so (extra -D defines) for A/B runs on the GPU box.

python tools/variant_build.py NAME:DEF1,DEF2 [NAME:...]   -> paper_2601_19911_b200/variants/NAME.so
Select one at run time with GOLP_B200_LIB=paper_2601_19911_b200/variants/NAME.so.
"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200.csrc import build  # noqa: E402

out_dir = build.PKG / "variants"
out_dir.mkdir(exist_ok=True)


def one(spec: str) -> str:
    name, _, defs = spec.partition(":")
    defines = [d for d in defs.split(",") if d]
    path = build.build(out=out_dir / f"{name}.so", defines=defines)
    log = (build.PKG / "build_ptxas.log").read_text()
    return f"{name}: {path}"


with ThreadPoolExecutor(4) as ex:
    for line in ex.map(one, sys.argv[1:]):
        print(line)
