#!/bin/bash
# rerank prefetch A/B + rerank phase profile + racecheck attribution
set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_scale_a.py tests/test_gpu_enn.py tests/test_gpu_two_phase.py tests/test_gpu_stream.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sel.txt
timeout 900 python bench.py --config 2 --no-cpu > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err; echo "cfg2 rc=$?"; cat $OUT/bench_cfg2.json
timeout 900 bash scripts/prof_rerank.sh $OUT/rr 2 > /dev/null 2>&1; echo "prof rc=$?"; cat $OUT/rr/phases.txt | tail -8
export VS_TC_PAIR=0
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_tc.py::test_tc_random_filtered -q -x -p no:cacheprovider > $OUT/racecheck_tc_single.txt 2>&1; echo "racecheck tc single-CTA rc=$?"; grep SUMMARY $OUT/racecheck_tc_single.txt
unset VS_TC_PAIR
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_enn.py::test_random_instances_match_reference_goldens tests/test_gpu_scale_a.py::test_config3_ivf_sampled_queries_equal_oracle -q -x -p no:cacheprovider > $OUT/racecheck_rerank.txt 2>&1; echo "racecheck rerank/ivf rc=$?"; grep -E "SUMMARY" $OUT/racecheck_rerank.txt; grep -A3 "Error\|Warning" $OUT/racecheck_rerank.txt | grep Thread | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head
