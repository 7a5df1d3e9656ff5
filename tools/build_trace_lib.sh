#!/bin/bash
# Diagnostics build of the backend with -DSP_CTA_TRACE (per-CTA start / end /
# staging times of k_score_flow, printed with SP_SCORE_TRACE=1) into
# build_trace/libsp_trace.so; load it with SP_LIB=build_trace/libsp_trace.so.
set -e
cd "$(dirname "$0")/.."
T=$(mktemp -d)
for f in fold search capi comm; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
    -Xcompiler -fPIC -Xcompiler -fno-fast-math --expt-relaxed-constexpr -DSP_CTA_TRACE \
    -c paper_2302_00247_b200/csrc/$f.cu -o $T/$f.o 2>/dev/null &
done
wait
g++ -O2 -std=c++17 -fPIC -c paper_2302_00247_b200/csrc/ingest.cpp -o $T/ingest.o
mkdir -p build_trace
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_trace/libsp_trace.so $T/*.o \
  -lcudart_static -lrt -lpthread -ldl
rm -rf $T
