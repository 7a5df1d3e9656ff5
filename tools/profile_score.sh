#!/bin/bash
# ncu --set full of the dominant kernel (k_score_flow<walk, pair>) on the c5
# bench workload, summarised into profiles/<name>.txt with the kernel's SASS
# sha256 in the header (bench.py uses the instruction count only while the
# built kernel is that binary).  Run on the GPU box:
#   tools/profile_score.sh r2_k_score_c5_walk
set -e
cd "$(dirname "$0")/.."
NAME=${1:-r2_k_score_c5_walk}
MODE=${2:-walk}
KREGEX=${3:-k_score_flow}
# the c5 search launches the residual group first: with k_score_flow it runs as k_search_small now (SKIP=0)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX}" --launch-skip ${SKIP:-0} -c 1 -f \
    -o gpurun_out/${NAME} python tools/ncu_target.py c5 ${MODE} 1 > gpurun_out/${NAME}.log 2>&1
SHA=$(python -c "import bench; print(bench.kernel_sass_sha())")
CANDS=$(python -c "import json; print(json.load(open('tests/golden/c5_full.json'))['candidates'])")
python tools/summarize_ncu.py gpurun_out/${NAME}.ncu-rep "${NAME}: c5 throughput tier, mode ${MODE}" \
    "sass_sha256: ${SHA}" > gpurun_out/${NAME}.txt
echo "# candidates: ${CANDS}" >> gpurun_out/${NAME}.txt
cat gpurun_out/${NAME}.txt
