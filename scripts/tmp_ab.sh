#!/bin/bash
set -u
OUT=gpurun_out/r2ae
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_enn.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_sel.txt
for pd in 4 2 1 0 8 4; do
  VS_RR_PD=$pd timeout 600 python bench.py --config 2 --no-cpu --steps 20 > $OUT/cfg2_pd$pd.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg2_pd$pd.json'));print('cfg2 pd=$pd', d['ms_per_step'], d['kernel_ms_per_step']['rerank'], d['clocks']['sm_mhz'])"
done
