#!/bin/bash
# new coarse select + list-unit filtered scan: tests, cfg3/cfg4 bench, ncu of the new kernels and of cfg2 k_rerank
set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_ivf_kernels.py tests/test_gpu_scale_a.py tests/test_gpu_tc.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sel.txt
for c in 3 4; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"; cat $OUT/bench_cfg$c.json; tail -2 $OUT/bench_cfg$c.err
done
bash scripts/ncu_cfg.sh r2e 3 "k_coarse_select k_ivf_scan_sel k_rerank"
bash scripts/ncu_cfg.sh r2e 2 "k_rerank"
du -sh $OUT
