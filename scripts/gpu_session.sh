#!/bin/bash
# One gpurun session: parity tests, the default bench line, the ncu launch
# list of the same command, and one full ncu capture of the top kernel.
# Usage (from the repo root on the GPU box): bash scripts/gpu_session.sh TAG [KERNEL_REGEX]
set -u
TAG=${1:-run}
KREGEX=${2:-k_enn_scan}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
tail -3 $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
cat $OUT/bench.json
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > $OUT/ncu_launch_bench.log 2>&1
  echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 \
      -o $OUT/prof python bench.py --steps 1 --warmup 1 --no-cpu > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
