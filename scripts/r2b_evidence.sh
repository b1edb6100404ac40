bash scripts/ncu_cfg.sh r2b 3 "k_ivf_scan_sel k_dense_select k_refine32 k_rerank k_enn_scan_tc"
bash scripts/ncu_cfg.sh r2b 2 "k_enn_scan_tc k_rerank k_stage_rows"
bash scripts/ncu_cfg.sh r2b 4 "k_enn_scan_tc"
bash scripts/r2_checks.sh r2b
