#!/bin/bash
set -u
OUT=gpurun_out/r2x
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ivf_kernels.py tests/test_gpu_ivf.py tests/test_gpu_scale_a.py tests/test_gpu_scale_b.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for c in 3 4; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/cfg$c.json 2> $OUT/cfg$c.err
  python -c "import json;d=json.load(open('$OUT/cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('e2e_host_ms_per_step'), d['kernel_ms_per_step'], d.get('ivf_survivors_per_query'))"
done
