#!/bin/bash
# Phase timing of the re-rank kernel (clock64 per phase, thread 0 of each CTA):
# builds a profiling variant of the library into /tmp and runs config-2 searches.
set -eu
OUT=${1:-gpurun_out/rr_phases}
mkdir -p $OUT /tmp/vsprof
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 -I include -DVS_RERANK_PROFILE ${PROF_FLAGS:-}"
for f in paper_2605_15957_b200/csrc/*.cu; do $NV -c $f -o /tmp/vsprof/$(basename $f).o & done; wait
$NV -shared -o /tmp/vsprof/libvsb200_prof.so /tmp/vsprof/*.o -lcuda
shift
VS_B200_LIB=/tmp/vsprof/libvsb200_prof.so python scripts/prof_rerank.py "${@:-2}" > $OUT/phases.txt 2>&1
cat $OUT/phases.txt
