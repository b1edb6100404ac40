#!/bin/bash
# fp16-operand A/B + cfg3 kernel evidence + racecheck details
set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_scale_a.py tests/test_gpu_ivf.py tests/test_gpu_enn.py tests/test_gpu_two_phase.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sel.txt
for c in 2 3; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c f16 rc=$?"; cat $OUT/bench_cfg$c.json
  VS_TC_BF16=1 timeout 900 python bench.py --config $c --no-cpu > $OUT/bench_cfg${c}_bf16.json 2> $OUT/bench_cfg${c}_bf16.err; echo "cfg$c bf16 rc=$?"; cat $OUT/bench_cfg${c}_bf16.json
done
bash scripts/ncu_cfg.sh r2c 3 "k_ivf_scan_sel k_dense_select k_refine32 k_rerank"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 python -m pytest tests/test_gpu_tc.py::test_tc_random_filtered -q -x -p no:cacheprovider > $OUT/racecheck_tc.txt 2>&1; echo "racecheck tc rc=$?"
grep -E "SUMMARY|Race reported|Error: Race|Warning: Race|at .*0x|in .*k_" $OUT/racecheck_tc.txt | sort | uniq -c | sort -rn | head -40
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 python -m pytest tests/test_gpu_ivf_kernels.py -q -x -p no:cacheprovider > $OUT/racecheck_ivf.txt 2>&1; echo "racecheck ivf rc=$?"
grep -E "SUMMARY|Race reported|Error: Race|Warning: Race|at .*0x|in .*k_" $OUT/racecheck_ivf.txt | sort | uniq -c | sort -rn | head -40
du -sh $OUT
