#!/bin/bash
# warp-per-query re-rank for small k: full gpu suite + configs 1/3/4
set -u
OUT=gpurun_out/r2n
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -x -m gpu > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.txt
for c in 3 1 4; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/cfg$c.json 2> $OUT/cfg$c.err
  python -c "import json;d=json.load(open('$OUT/cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])"
  grep check $OUT/cfg$c.err | tail -1
done
VS_RR_WARP=0 timeout 900 python bench.py --config 3 --no-cpu > $OUT/cfg3_nowarp.json 2>/dev/null
python -c "import json;d=json.load(open('$OUT/cfg3_nowarp.json'));print('cfg3 no-warp', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
