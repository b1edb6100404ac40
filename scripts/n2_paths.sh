#!/bin/bash
# The N > 1 bench code paths on ONE GPU (torchrun, 2 ranks on cuda:0, gloo;
# VS_BENCH_ONE_GPU=1) for configs 2, 3, 4, 5 and the reference arm. Code-path
# evidence only: reduced collections (--n-rows), never reported numbers.
# Usage: bash scripts/n2_paths.sh TAG
set -u
OUT=gpurun_out/${1:-n2}
mkdir -p $OUT
port=29621
for c in 2 3 4 5; do
  rows=$([ $c = 4 ] && echo 4000000 || echo 2000000)
  VS_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port $port bench.py --gpus 2 --config $c --n-rows $rows \
      --steps 3 --warmup 3 --no-cpu > $OUT/n2_cfg$c.json 2> $OUT/n2_cfg$c.err
  echo "N=2 cfg$c rc=$?"; port=$((port + 1))
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $port bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > $OUT/n2_ref.json 2> $OUT/n2_ref.err
echo "N=2 reference rc=$?"
