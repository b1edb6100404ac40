#!/bin/bash
set -u
OUT=gpurun_out/r2s
mkdir -p $OUT
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:k_enn_scan_tc -c 1 \
    -o $OUT/prof_a python bench.py --config 2 --steps 1 --warmup 1 --no-cpu > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof_a.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/prof_cfg2_k_enn_scan_tc_source.csv.gz
ncu -i $OUT/prof_a.ncu-rep --page raw --csv > $OUT/prof_cfg2_k_enn_scan_tc_raw.csv 2>/dev/null
rm -f $OUT/prof_a.ncu-rep
ls -la $OUT
