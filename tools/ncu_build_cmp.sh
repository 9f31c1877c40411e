#!/bin/bash
# Warm-cache per-kernel times of the C2 build for library variants (GPU box).
for v in "$@"; do
  GOLP_B200_LIB=paper_2601_19911_b200/variants/lib_$v.so ncu --metrics gpu__time_duration.sum --clock-control none \
    --cache-control none -k regex:"part_|join_|scan_" --csv python tools/join_breakdown.py 1e6 1e7 2e6 2 \
    > gpurun_out/ncu_build_$v.csv 2>&1
done
