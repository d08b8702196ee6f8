#!/bin/bash
# functional check of the N>1 bench path on ONE GPU (gloo collectives, all ranks on cuda:0):
# 2 and 3 ranks sequence-sharded, 4 ranks as 2 head groups x 2 sequence shards
mkdir -p gpurun_out
: > gpurun_out/multirank.log
run() {
  echo "== $*" >> gpurun_out/multirank.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $1 --steps 2 --warmup 3 --context 65536 --dist-backend gloo --one-gpu "${@:2}" >> gpurun_out/multirank.log 2>&1
  echo "rc=$?" >> gpurun_out/multirank.log
}
run 2
run 3
run 4 --head-groups 2
echo "== single c4-shape ctx 65536" >> gpurun_out/multirank.log
timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --context 65536 >> gpurun_out/multirank.log 2>&1
