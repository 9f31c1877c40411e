#!/bin/bash
# Warm-cache per-kernel times of one C4-shaped span (build 1e8, 2^30 probes) (GPU box).
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
  -k regex:"part_|join_|scan_" --csv python tools/join_breakdown.py 1e8 1073741824 2e8 1 \
  > gpurun_out/ncu_c4_span.csv 2>&1
