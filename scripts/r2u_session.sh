#!/bin/bash
set -u
OUT=gpurun_out/r2u
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_enn.py tests/test_gpu_scale_a.py tests/test_gpu_two_phase.py tests/test_gpu_stream.py tests/test_gpu_scale_c.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for c in 2 5 1; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/cfg$c.json 2> $OUT/cfg$c.err
  python -c "import json;d=json.load(open('$OUT/cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['kernel_ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
  grep check $OUT/cfg$c.err | tail -1
done
timeout 900 python scripts/emulate_shards.py 2 4 8 > $OUT/emulate.txt 2>&1; grep '^{' $OUT/emulate.txt
