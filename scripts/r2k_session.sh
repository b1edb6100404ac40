#!/bin/bash
# staggered phase-A compactions: parity + A/B on config 2 and the 8-shard emulation
set -u
OUT=gpurun_out/r2k
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_enn.py tests/test_gpu_scale_a.py::test_config2_sampled_queries_equal_oracle tests/test_gpu_two_phase.py tests/test_gpu_ivf_kernels.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for st in 2 0 2 0 1 4; do
  VS_TC_STAGGER=$st VS_TC_DEBUG=1 timeout 600 python bench.py --config 2 --no-cpu --steps 10 > $OUT/cfg2_st$st.json 2> $OUT/cfg2_st$st.err
  python -c "import json;d=json.load(open('$OUT/cfg2_st$st.json'));print('cfg2 stagger=$st', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
  grep "vs_tc\]" $OUT/cfg2_st$st.err | tail -1 | sed 's/.*mma wait-full/mma wait-full/' | cut -c1-150
done
timeout 900 python scripts/emulate_shards.py 8 > $OUT/emulate8.jsonl 2>&1; grep '^{' $OUT/emulate8.jsonl
