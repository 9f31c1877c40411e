"""One resident Top-K over N uniform keys (tools/, for ncu captures).
python tools/topk_resident.py N K [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_19911_b200 import resident  # noqa: E402

n, k = int(float(sys.argv[1])), int(float(sys.argv[2]))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = torch.Generator(device="cuda").manual_seed(7)
keys = torch.randint(0, 2**53, (n,), device="cuda", generator=g, dtype=torch.int64).double()
rows = torch.arange(n, dtype=torch.int32, device="cuda")
for _ in range(reps):
    out, _ = resident.topk(keys, rows, k)
torch.cuda.synchronize()
print("ok", out[:4].tolist())
