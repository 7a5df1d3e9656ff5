#!/bin/bash
# Every BASELINE config through bench.py on one GPU (SURVEY 8(d) "per config"):
#   tools/all_configs.sh [out.jsonl]
out=${1:-gpurun_out/configs.jsonl}
: > "$out"
for w in c1 c2 c3 c3_slow c4 c4_2x4 c4_2x4_slow; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --cpu-seconds 3 --no-python-reference \
    --no-fold-roofline >> "$out" || echo "{\"workload\": \"$w\", \"failed\": true}" >> "$out"
done
