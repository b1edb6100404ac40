#!/bin/bash
# split phase B (select kernel at 5 CTAs/SM + score/top-k kernel): parity + A/B
set -u
OUT=gpurun_out/r2g
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -x -m gpu > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.txt
for v in "1 2" "0 2" "1 3" "0 3" "1 2" "0 2"; do
  set -- $v
  VS_RR_SPLIT=$1 timeout 600 python bench.py --config $2 --no-cpu --steps 20 > $OUT/cfg$2_split$1.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg$2_split$1.json'));print('cfg$2 split=$1', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
done
