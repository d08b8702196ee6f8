#!/bin/bash
# One GPU call: the GPU parity suite, the default bench line, a gloo two-rank
# functional run of the sharded bench path (one GPU), logs into gpurun_out/.
set -x
OUT=gpurun_out/${TAG:-run}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
if [ -n "$MULTI" ]; then
  timeout 900 python bench.py --gpus 2 --one-gpu --dist-backend gloo --context 131072 --steps 3 --warmup 3 > $OUT/multi.log 2>&1; echo "multi rc=$?" >> $OUT/multi.log
fi
tail -3 $OUT/pytest.log; tail -2 $OUT/bench.log; tail -2 $OUT/multi.log 2>/dev/null
