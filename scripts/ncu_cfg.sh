#!/bin/bash
# ncu launch list + one --set full capture per kernel regex for one bench config.
# The .ncu-rep files are reduced on the box to raw/details CSVs (gpurun brings
# back at most 64 MiB); set KEEP_REP=1 to keep the report itself.
# Usage: bash scripts/ncu_cfg.sh TAG CONFIG "regex1 regex2 ..." [extra bench args]
set -u
TAG=$1; CFG=$2; REGEXES=${3:-}; EXTRA=${4:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_cfg$CFG.csv python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu $EXTRA \
    > $OUT/ncu_launch_cfg$CFG.log 2>&1
echo "ncu launches cfg$CFG rc=$?"
for R in $REGEXES; do
  REP=$OUT/prof_cfg${CFG}_$R
  timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:$R -c 1 \
      -o $REP python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu $EXTRA \
      > $OUT/ncu_full_cfg${CFG}_$R.log 2>&1
  echo "ncu full cfg$CFG $R rc=$?"
  if [ -f $REP.ncu-rep ]; then
    ncu -i $REP.ncu-rep --page raw --csv > ${REP}_raw.csv 2>/dev/null
    ncu -i $REP.ncu-rep --page details --csv > ${REP}_details.csv 2>/dev/null
    ncu -i $REP.ncu-rep --page source --csv > ${REP}_source.csv 2>/dev/null
    gzip -f ${REP}_source.csv
    [ "${KEEP_REP:-0}" = "1" ] || rm -f $REP.ncu-rep
  fi
done
