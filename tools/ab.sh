#!/bin/bash
# A/B kernel timing on the GPU box: tools/ab.sh lib1.so lib2.so ...  (modes: walk skip)
for l in "$@"; do SP_LIB=$l timeout 200 python tools/kbench.py walk skip; done
for l in "$@"; do
  SP_LIB=$l timeout 300 ncu --metrics smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum \
    --clock-control none -k regex:k_score -s 1 -c 1 python tools/ncu_target.py c5 walk 2 2>&1 | grep -E "k_score|inst_executed|issue_active|duration" | sed "s|^|$l |"
done
