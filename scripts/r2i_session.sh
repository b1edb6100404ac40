#!/bin/bash
# round-2 evidence: bench lines for all configs + reference arm, launch lists, ncu captures of the top kernels
set -u
OUT=gpurun_out/r2i
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu.txt 2>&1
for c in 2 1 3 4 5; do
  timeout 1500 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err; echo "cfg$c rc=$?"
  python -c "import json;d=json.load(open('$OUT/bench_cfg$c.json'));print('cfg$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['kernel_ms_per_step'], d['clocks'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"; cat $OUT/bench_reference.json
bash scripts/ncu_cfg.sh r2i 2 "k_enn_scan_tc"
bash scripts/ncu_cfg.sh r2i 3 "k_ivf_scan_sel k_enn_scan_tc"
bash scripts/ncu_cfg.sh r2i 4 "k_enn_scan_tc"
rm -f $OUT/*_source.csv.gz
du -sh $OUT
