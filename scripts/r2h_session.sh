#!/bin/bash
# narrow rerank single-row scorer (no spills) + phase-A stall counters + ncu of the split score kernel
set -u
OUT=gpurun_out/r2h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_enn.py tests/test_gpu_ivf.py tests/test_gpu_tc.py tests/test_gpu_scale_a.py tests/test_gpu_wide.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for c in 3 1; do
  timeout 600 python bench.py --config $c --no-cpu > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
  python -c "import json;d=json.load(open('$OUT/bench_cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
done
VS_TC_DEBUG=1 timeout 600 python bench.py --config 2 --no-cpu --steps 3 --warmup 3 > $OUT/cfg2_dbg.json 2> $OUT/cfg2_dbg.err; grep "vs_tc\]" $OUT/cfg2_dbg.err | tail -3
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:k_rerank -s 1 -c 1 \
    -o $OUT/prof_cfg2_rerank_ph2 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu > $OUT/ncu_ph2.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof_cfg2_rerank_ph2.ncu-rep --page raw --csv > $OUT/prof_cfg2_rerank_ph2_raw.csv 2>/dev/null
ncu -i $OUT/prof_cfg2_rerank_ph2.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/prof_cfg2_rerank_ph2_source.csv.gz
rm -f $OUT/prof_cfg2_rerank_ph2.ncu-rep
