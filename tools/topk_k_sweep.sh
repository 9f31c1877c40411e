#!/bin/bash
# C3 K=1e5 resident step time per library variant (GPU box): tools/topk_k_sweep.sh v1 v2 ...
for v in "$@"; do
  GOLP_B200_LIB=paper_2601_19911_b200/variants/lib_$v.so timeout 300 python bench.py --workload topk_c3 --k 100000 \
    --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'])"
done
