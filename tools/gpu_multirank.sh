#!/bin/bash
# functional check of the N>1 bench path on ONE GPU: 2 and 3 ranks on cuda:0, gloo collectives
mkdir -p gpurun_out
: > gpurun_out/multirank.log
for n in 2 3; do
  echo "== ranks $n" >> gpurun_out/multirank.log
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $n --steps 2 --warmup 3 --context 65536 --dist-backend gloo --one-gpu >> gpurun_out/multirank.log 2>&1
  echo "rc=$?" >> gpurun_out/multirank.log
done
echo "== single c4-shape ctx 65536" >> gpurun_out/multirank.log
timeout 300 python bench.py --config c4 --steps 2 --warmup 3 --context 65536 >> gpurun_out/multirank.log 2>&1
