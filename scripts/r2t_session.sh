#!/bin/bash
# sampled admission-bound seed for phase A (VS_TC_TAU_SAMPLE)
set -u
OUT=gpurun_out/r2t
mkdir -p $OUT
VS_TC_TAU_SAMPLE=8192 timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_enn.py tests/test_gpu_scale_a.py::test_config2_sampled_queries_equal_oracle tests/test_gpu_two_phase.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
for ts in 0 8192 32768 0 8192; do
  VS_TC_TAU_SAMPLE=$ts VS_TC_DEBUG=1 timeout 600 python bench.py --config 2 --no-cpu --steps 10 > $OUT/cfg2_ts$ts.json 2> $OUT/cfg2_ts$ts.err
  python -c "import json;d=json.load(open('$OUT/cfg2_ts$ts.json'));print('cfg2 ts=$ts', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'], d['overflow_requeries_total'])"
  grep "vs_tc\]" $OUT/cfg2_ts$ts.err | tail -1 | sed 's/.*mma wait-full/mma wait-full/' | cut -c1-160
done
for ts in 8192 32768; do
  VS_TC_TAU_SAMPLE=$ts timeout 900 python scripts/emulate_shards.py 8 > $OUT/emu8_ts$ts.txt 2>&1; echo "emu8 ts=$ts"; grep '^{' $OUT/emu8_ts$ts.txt
done
