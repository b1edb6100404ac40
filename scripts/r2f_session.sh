#!/bin/bash
# restored filtered scan (division-free) + fp64 pipe rates + cfg2 A/B (fp16/bf16 operands, rerank build)
set -u
OUT=gpurun_out/r2f
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_rates scripts/micro/fp64_rates.cu && /tmp/fp64_rates > $OUT/fp64_rates.txt 2>&1; cat $OUT/fp64_rates.txt
timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_ivf_kernels.py tests/test_gpu_scale_a.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
timeout 900 python bench.py --config 3 --no-cpu > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err; echo "cfg3 rc=$?"; python -c "import json;d=json.load(open('$OUT/bench_cfg3.json'));print(d['ms_per_step'],d['kernel_ms_per_step'])"
i=0
for v in "f16 -1" "f16 0" "bf16 -1" "f16 -1" "bf16 -1" "f16 0"; do
  set -- $v; i=$((i+1))
  if [ $1 = bf16 ]; then export VS_TC_BF16=1; else unset VS_TC_BF16; fi
  VS_RR_WIDE=$2 timeout 600 python bench.py --config 2 --no-cpu --steps 20 > $OUT/cfg2_$i.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg2_$i.json'));print('$1 wide=$2', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'], d.get('survivors_per_query'))"
done
