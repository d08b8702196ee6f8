#!/bin/bash
# capture kernel iteration: pipeline tests, c2 bench line, ncu of the capture stage
OUT=${OUT:-gpurun_out/${TAG:-cap}}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_measured.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras ${BENCH} > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include sts.capture/ -c 2 -o $OUT/cap -f python bench.py --eager --steps 1 --warmup 1 --no-cpu-baseline --no-extras --parity-units 0 ${BENCH} > $OUT/ncu.log 2>&1
tail -3 $OUT/pytest.log; python - <<'PY'
import json,os
t=open(os.environ.get("OUT","gpurun_out/cap")+"/bench.log").read().splitlines()
for l in t:
    if l.startswith("{"):
        d=json.loads(l); print("attend",d["value"],"capture",d["mask_build_us"],"parity",d.get("parity",{}).get("masks_bit_exact"))
PY
