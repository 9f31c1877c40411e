#!/bin/bash
# Launch lists and the changed kernel's full capture for profiles/ (GPU box).
set -u
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_join_c2.csv 2>&1
echo c2 rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"part_|join_|scan_" --csv python tools/join_breakdown.py 1e8 1073741824 2e8 1 \
  > gpurun_out/launches_join_c4_partitioned.csv 2>&1
echo c4 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"join_probe_part_kernel" -c 1 \
  -o gpurun_out/full_c4span_probe_part python tools/join_breakdown.py 1e8 268435456 2e8 1 > gpurun_out/full_c4span.log 2>&1
echo full rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|filter|topk|rank" --csv \
  python bench.py --workload topk_c1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_topk_c1_fused.csv 2>&1
echo c1 rc=$?
