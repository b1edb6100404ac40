#!/bin/bash
# whole-list filtered scan (v4) + phase-A split-count sweep + shard emulation
set -u
OUT=gpurun_out/r2j
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_ivf_kernels.py tests/test_gpu_scale_a.py tests/test_gpu_wide.py -q -x > $OUT/pytest_sel.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_sel.txt
timeout 600 python bench.py --config 3 --no-cpu > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err
python -c "import json;d=json.load(open('$OUT/bench_cfg3.json'));print('cfg3', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])"
for ns in 11 22 33; do
  VS_TC_NSPLIT=$ns timeout 600 python bench.py --config 2 --no-cpu --steps 10 > $OUT/cfg2_ns$ns.json 2>/dev/null
  python -c "import json;d=json.load(open('$OUT/cfg2_ns$ns.json'));print('cfg2 nsplit=$ns', d['ms_per_step'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
done
timeout 900 python scripts/emulate_shards.py 2 4 8 > $OUT/emulate_shards.jsonl 2>&1; cat $OUT/emulate_shards.jsonl | grep '^{'
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ivf_scan_sel -c 2 --csv \
    --log-file $OUT/scan_cfg3.csv python bench.py --config 3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; grep -E "duration|dram" $OUT/scan_cfg3.csv | tail -3
