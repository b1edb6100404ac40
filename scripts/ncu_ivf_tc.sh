#!/bin/bash
# ncu evidence for the config-4 IVF tensor-core list scan (k_enn_scan_tc<.., 2, ..>):
# launch list of the timed region + one --set full capture of the scan.
# Usage: bash scripts/ncu_ivf_tc.sh TAG
set -u
TAG=${1:-ivf}
OUT=gpurun_out/$TAG
mkdir -p $OUT
[ -n "${SKIP_LAUNCHES:-}" ] || timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_cfg4.csv python bench.py --config 4 --steps 2 --warmup 1 --no-cpu \
    > $OUT/ncu_launch_cfg4.log 2>&1
echo "ncu launches cfg4 rc=$?"
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
    --kernel-name-base demangled -k "regex:bn256::tc::k_enn_scan_tc" -c 1 -o $OUT/prof_cfg4_mode2 \
    python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > $OUT/ncu_full_cfg4_mode2.log 2>&1
echo "ncu full cfg4 mode2 rc=$?"
