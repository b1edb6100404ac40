#!/bin/bash
# compute-sanitizer over the kernels changed late in round 2: the filtered
# tensor-core IVF scan (norm-load hoist), the bitmap permutation, the re-rank
# flat gather, fp16 shadow staging, pinned-output transfers.
set -u
OUT=gpurun_out/${1:-san_late}
mkdir -p $OUT
SEL="tests/test_gpu_ivf_kernels.py tests/test_gpu_tc.py::test_tc_f16_shadow_repeated_searches_and_mutation tests/test_gpu_enn.py::test_large_pinned_host_outputs_staged"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest $SEL -q -x -p no:cacheprovider > $OUT/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_$tool.txt
  tail -4 $OUT/sanitizer_$tool.txt
done
