#!/bin/bash
# ncu launch list + one --set full capture per kernel regex for one bench config.
# Usage: bash scripts/ncu_cfg.sh TAG CONFIG "regex1 regex2 ..."
set -u
TAG=$1; CFG=$2; REGEXES=${3:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_cfg$CFG.csv python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu \
    > $OUT/ncu_launch_cfg$CFG.log 2>&1
echo "ncu launches cfg$CFG rc=$?"
for R in $REGEXES; do
  timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:$R -c 1 \
      -o $OUT/prof_cfg${CFG}_$R python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu \
      > $OUT/ncu_full_cfg${CFG}_$R.log 2>&1
  echo "ncu full cfg$CFG $R rc=$?"
done
