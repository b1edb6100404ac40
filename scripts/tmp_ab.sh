#!/bin/bash
set -u
OUT=gpurun_out/r2ah
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ivf_build.py tests/test_gpu_ivf_kernels.py tests/test_gpu_ivf.py -q -x -s > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt; grep -i "agreement" $OUT/pytest_sel.txt
timeout 900 python bench.py --config 3 --no-cpu --steps 5 > $OUT/cfg3.json 2> $OUT/cfg3.err; grep -E "build" $OUT/cfg3.err | head -2
timeout 1200 python bench.py --config 4 --no-cpu --steps 5 > $OUT/cfg4.json 2> $OUT/cfg4.err; grep -E "build" $OUT/cfg4.err | head -2
