#!/bin/bash
# quick iteration: selected GPU tests + one short bench line (each under its own timeout)
OUT=gpurun_out/${TAG:-q}
mkdir -p $OUT
timeout ${TT:-600} python -m pytest ${TESTS:-tests/test_gpu_pipeline.py} -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
if [ -n "$BENCH" ]; then timeout 600 python bench.py $BENCH > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log; fi
tail -15 $OUT/pytest.log; tail -3 $OUT/bench.log 2>/dev/null | cut -c1-1500
