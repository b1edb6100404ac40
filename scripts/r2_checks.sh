#!/bin/bash
# Round-2 hardening evidence on one GPU: compute-sanitizer (memcheck, racecheck,
# synccheck) over the tensor-core phase A, the re-rank, the IVF scans and the
# large-k' path; the N > 1 bench code paths (torchrun, 2 ranks on cuda:0,
# gloo) for configs 2 and 4; the shard emulation of config 2.
# Usage: bash scripts/r2_checks.sh TAG
set -u
TAG=${1:-r2checks}
OUT=gpurun_out/$TAG
mkdir -p $OUT
SEL="tests/test_gpu_tc.py::test_tc_random_filtered tests/test_gpu_ivf.py::test_coarse_quantizer_modes_equal_oracle tests/test_gpu_ivf_kernels.py tests/test_gpu_wide.py::test_ivf_large_k_equals_oracle tests/test_gpu_wide.py::test_enn_large_k_equals_oracle"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest $SEL -q -x -p no:cacheprovider > $OUT/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> $OUT/sanitizer_$tool.txt
  tail -4 $OUT/sanitizer_$tool.txt
done
for c in 2 4; do
  rows=$([ $c = 4 ] && echo 4000000 || echo 2000000)
  VS_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --config $c --n-rows $rows \
      --steps 3 --warmup 3 --no-cpu > $OUT/n2_cfg$c.json 2> $OUT/n2_cfg$c.err
  echo "N=2 cfg$c rc=$?"; cat $OUT/n2_cfg$c.json; tail -2 $OUT/n2_cfg$c.err
done
timeout 900 python scripts/emulate_shards.py 2 4 8 > $OUT/emulate_shards.jsonl 2>&1; cat $OUT/emulate_shards.jsonl
