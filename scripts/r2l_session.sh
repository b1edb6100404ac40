#!/bin/bash
# filtered tensor-core IVF scan (mma.sync): parity + config 3 A/B + ncu
set -u
OUT=gpurun_out/r2l
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ivf_kernels.py tests/test_gpu_ivf.py tests/test_gpu_scale_a.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_sel.txt
for m in 1 0 1; do
  VS_IVF_MMA=$m timeout 600 python bench.py --config 3 --no-cpu > $OUT/cfg3_mma$m.json 2> $OUT/cfg3_mma$m.err
  python -c "import json;d=json.load(open('$OUT/cfg3_mma$m.json'));print('cfg3 mma=$m', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])"
  tail -1 $OUT/cfg3_mma$m.err
done
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:k_ivf_scan_mma -c 1 \
    -o $OUT/prof_mma python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $OUT/prof_mma.ncu-rep --page raw --csv > $OUT/prof_cfg3_k_ivf_scan_mma_raw.csv 2>/dev/null
ncu -i $OUT/prof_mma.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/prof_cfg3_k_ivf_scan_mma_source.csv.gz
rm -f $OUT/prof_mma.ncu-rep
