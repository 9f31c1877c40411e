#!/bin/bash
# Round-2 measurement evidence for profiles/ (run on the GPU box; outputs in gpurun_out/r2_*).
#   bench lines of every config, launch lists, and the ncu captures behind roofline.traffic.
set -u
mkdir -p gpurun_out
B=gpurun_out/r2_bench_lines.jsonl
: > $B
run() { python bench.py "$@" 2>>gpurun_out/r2_bench.err | tail -1 >> $B; echo "bench $* rc=${PIPESTATUS[0]}"; }
run
run --workload topk_c1
run --workload topk_c3 --k 10 --steps 10
run --workload topk_c3 --k 1000 --steps 10
run --workload topk_c3 --k 100000 --steps 10
run --workload join_c4 --steps 5
run --probe-positions
run --workload join_c4 --steps 5 --probe-positions
run --workload topk_c3 --k 1000 --dist zipf_hi --steps 10 --row-column
run --workload topk_c3 --k 1000 --dist zipf_hi --steps 10
run --workload topk_c3 --k 1000 --dist zipf_lo --steps 10
# launch list of the default bench command (cold-cache, serialized: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-verify > gpurun_out/r2_launches_join_c2.csv 2>&1
echo "c2 launches rc=$?"
# C2 probe / build kernels, full sets (DRAM traffic per launch for roofline.traffic)
ncu --set full --clock-control none --import-source on -k regex:"join_match_kernel|join_emit_kernel|join_insert|join_finalize" \
  -s 7 -c 4 -o gpurun_out/r2_full_join_c2 python tools/join_breakdown.py 1e6 1e7 2e6 3 > gpurun_out/r2_full_join_c2.log 2>&1
echo "c2 full rc=$?"
# the same kernels without ncu's cache flush (--cache-control none): the state the bench's
# step sees (the table was just built and sits in L2); bench.py's roofline.traffic uses these
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"join_match_kernel|join_emit_kernel" \
  -s 4 -c 2 -o gpurun_out/r2_full_join_c2_warm python tools/join_breakdown.py 1e6 1e7 2e6 3 > gpurun_out/r2_full_join_c2_warm.log 2>&1
echo "c2 warm rc=$?"
# C4: every probe-phase kernel of one whole 1e8 x 2e9 join, time + DRAM bytes
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"part_|join_|scan_" python tools/join_breakdown.py 1e8 2e9 2e8 1 > gpurun_out/r2_launches_join_c4.csv 2>&1
echo "c4 launches rc=$?"
# C1 fused Top-K and the C3 filter
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"select|filter|topk|rank" python bench.py --workload topk_c1 --steps 3 --warmup 3 --no-cpu-baseline --no-verify \
  > gpurun_out/r2_launches_topk_c1.csv 2>&1
echo "c1 launches rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"topk_filter" -c 2 python tools/topk_resident.py 1e9 1000 2 > gpurun_out/r2_launches_topk_c3_filter.csv 2>&1
echo "c3 filter rc=$?"
