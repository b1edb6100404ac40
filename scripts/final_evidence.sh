#!/bin/bash
# round-2 final evidence: full gpu suite, smoke, all configs, reference arm, launch lists
set -u
OUT=gpurun_out/final
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x --durations=10 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['kernel_ms_per_step'], d['clocks']['sm_mhz'])"
  grep check $OUT/bench_cfg$c.err | tail -1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"; cat $OUT/bench_reference.json
for c in 2 3 4; do
  timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
      --log-file $OUT/launches_cfg$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1; echo "launches cfg$c rc=$?"
done
du -sh $OUT
