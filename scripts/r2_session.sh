#!/bin/bash
# Round-2 evidence session on one GPU: the gpu test suite, smoke(), bench lines
# for every config (1-5) and the reference arm for the default config.
# Usage: bash scripts/r2_session.sh TAG "1 2 3 4 5"
set -u
TAG=${1:-r2}
CFGS=${2:-"2 1 3 4 5"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
  tail -22 $OUT/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
fi
for c in $CFGS; do
  timeout 1500 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
  cat $OUT/bench_cfg$c.json; tail -2 $OUT/bench_cfg$c.err
done
if [ "${SKIP_REF:-0}" != "1" ]; then
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
  cat $OUT/bench_ref.json
fi
