#!/bin/bash
# Every bench line of the round (C2 default, C1, C3 x K, C3 Zipf-hi, C4), one JSON
# line each into gpurun_out/bench_lines.jsonl; logs beside it. Run on the GPU box.
set -u
mkdir -p gpurun_out
out=gpurun_out/bench_lines.jsonl
: > "$out"
run() {
  local tag=$1; shift
  timeout 900 python bench.py "$@" > "gpurun_out/bench_$tag.log" 2>&1
  echo "$tag rc=$?"
  tail -1 "gpurun_out/bench_$tag.log" | grep '^{' >> "$out"
}
run c2
run c1 --workload topk_c1
run c3_k10 --workload topk_c3 --k 10
run c3_k1000 --workload topk_c3 --k 1000
run c3_k100000 --workload topk_c3 --k 100000
run c3_zipfhi --workload topk_c3 --k 1000 --dist zipf_hi --no-cpu-baseline
run c3_zipflo --workload topk_c3 --k 1000 --dist zipf_lo --no-cpu-baseline
run c4 --workload join_c4
