#!/bin/bash
# ncu --set full of the hash-fold kernels on a 9.8M-node fold (tools/fold_scale.py),
# summarised into gpurun_out/<name>_<kernel>.txt.  Run on the GPU box.
set -e
cd "$(dirname "$0")/.."
NAME=${1:-r2_fold}
LAYERS=${2:-700000}
shift 2 || true
KERNELS=${@:-k_hg_prep k_hg_insert k_hg_verify k_hg_entry}
mkdir -p gpurun_out
for K in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k "regex:${K}\$" --launch-skip ${SKIP:-0} -c 1 -f \
      -o gpurun_out/${NAME}_${K} python tools/fold_scale.py --layers ${LAYERS} --reps 1 > /dev/null 2>&1
  python tools/summarize_ncu.py gpurun_out/${NAME}_${K}.ncu-rep "${NAME}: ${K}, ${LAYERS}-layer fold" > gpurun_out/${NAME}_${K}.txt
done
