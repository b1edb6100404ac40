#!/bin/bash
# End-of-round evidence: GPU tests, smoke, every bench config (with CPU
# baselines), ncu launch lists + full captures of the config-2 phase A and
# the config-4 list scan. Usage: bash scripts/r1_final.sh TAG
set -u
TAG=${1:-r1final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
SKIP_NCU=1 bash scripts/r1c_session.sh $TAG
bash scripts/ncu_cfg.sh $TAG 2 "k_enn_scan_tc k_rerank"
bash scripts/ncu_ivf_tc.sh $TAG
