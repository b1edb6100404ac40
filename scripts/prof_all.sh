#!/bin/bash
# ncu evidence for every bench config's hot kernels (launch lists of the timed
# region + one --set full capture each). Usage: bash scripts/prof_all.sh TAG
set -u
TAG=${1:-prof}
bash scripts/ncu_cfg.sh $TAG 2 "k_enn_scan_tc k_rerank"
bash scripts/ncu_cfg.sh $TAG 3 "k_ivf_scan_lmajor k_enn_scan_tc"
bash scripts/ncu_cfg.sh $TAG 4 "k_enn_scan_tc"
bash scripts/ncu_cfg.sh $TAG 1 "k_rerank"
