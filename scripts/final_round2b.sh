#!/bin/bash
# Round-2b evidence pass (run under gpurun, one GPU): compute-sanitizer over small invocations of
# every kernel, and the bench lines of the other workloads (c2 / c3 / c5) and the --bounds run.
mkdir -p gpurun_out/r2b
S=/usr/local/cuda/bin/compute-sanitizer
{
  for tool in memcheck synccheck racecheck; do
    echo "== $tool"
    timeout 900 $S --tool $tool python scripts/sanitize_small.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Race reported|Read access at|Write access at" | sort | uniq -c | sort -rn | head -40
  done
} > gpurun_out/r2b/sanitizer.txt 2>&1
for c in c2 c3 c5; do timeout 900 python bench.py --config $c > gpurun_out/r2b/bench_$c.json 2>/dev/null; done
timeout 900 python bench.py --bounds > gpurun_out/r2b/bench_bounds.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2b/bench_reference.json 2>/dev/null
ls -la gpurun_out/r2b
