#!/bin/bash
set -u
OUT=gpurun_out/r2r
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_enn.py tests/test_gpu_ivf_kernels.py tests/test_gpu_stream.py tests/test_gpu_output.py tests/test_gpu_two_phase.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_sel.txt
for z in 1 0 1; do
  VS_ZERO_COPY_OUT=$z timeout 600 python bench.py --config 2 --no-cpu --steps 10 > $OUT/cfg2_zc$z.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg2_zc$z.json'));print('cfg2 zc=$z', d['value'], d['e2e']['value'], d['ms_per_step'], d.get('e2e_host_ms_per_step'), d['e2e_kernel_ms_per_step'])"
done
VS_ZERO_COPY_OUT=1 timeout 600 python bench.py --config 3 --no-cpu > $OUT/cfg3.json 2>/dev/null
python -c "import json;d=json.load(open('$OUT/cfg3.json'));print('cfg3', d['value'], d['e2e']['value'], d['ms_per_step'], d.get('e2e_host_ms_per_step'))"
