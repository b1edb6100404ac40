#!/bin/bash
set -u
OUT=gpurun_out/r2y
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_two_phase.py tests/test_gpu_scale_a.py tests/test_gpu_group.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
timeout 600 python bench.py --config 2 --no-cpu --steps 20 > $OUT/cfg2.json 2>/dev/null
python -c "import json;d=json.load(open('$OUT/cfg2.json'));print('cfg2', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
timeout 900 python scripts/emulate_shards.py 2 4 8 > $OUT/emulate.txt 2>&1; grep '^{' $OUT/emulate.txt
