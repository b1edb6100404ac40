#!/bin/bash
# scaling: per-item cost in the phase-A split choice, k-th pass on the select kernel
set -u
OUT=gpurun_out/r2p
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_two_phase.py tests/test_gpu_tc.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for ic in 0 8 24; do
  VS_TC_ITEM_COST=$ic VS_TC_DEBUG=1 timeout 900 python scripts/emulate_shards.py 8 > $OUT/emu8_ic$ic.txt 2>&1
  echo "item_cost=$ic"; grep '^{' $OUT/emu8_ic$ic.txt; grep "vs_tc\]" $OUT/emu8_ic$ic.txt | head -1 | cut -c1-60
  VS_TC_ITEM_COST=$ic timeout 600 python bench.py --config 2 --no-cpu --steps 10 > $OUT/cfg2_ic$ic.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg2_ic$ic.json'));print('cfg2 ic=$ic', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
done
