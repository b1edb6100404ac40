#!/bin/bash
# Extra bench configs + the gpu tests of the IVF path.
# Usage: bash scripts/bench_cfgs.sh TAG "1 3"
set -u
TAG=${1:-cfgs}
CFGS=${2:-"1 3"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in $CFGS; do
  timeout 1500 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
  cat $OUT/bench_cfg$c.json; tail -3 $OUT/bench_cfg$c.err
done
