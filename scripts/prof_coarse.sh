#!/bin/bash
# Phase timing of the coarse-quantizer re-rank (profiling build, see prof_rerank.sh).
set -eu
OUT=${1:-gpurun_out/rr_coarse}
mkdir -p $OUT /tmp/vsprof
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177 -I include -DVS_RERANK_PROFILE"
for f in paper_2605_15957_b200/csrc/*.cu; do $NV -c $f -o /tmp/vsprof/$(basename $f).o & done; wait
$NV -shared -o /tmp/vsprof/libvsb200_prof.so /tmp/vsprof/*.o -lcuda
VS_B200_LIB=/tmp/vsprof/libvsb200_prof.so python scripts/coarse_probe.py 2000000 32 > $OUT/coarse_phases.json 2>&1
VS_B200_LIB=/tmp/vsprof/libvsb200_prof.so python scripts/prof_rerank.py 1 > $OUT/cfg1_phases.txt 2>&1
cat $OUT/coarse_phases.json $OUT/cfg1_phases.txt
