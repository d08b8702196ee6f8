mkdir -p gpurun_out/sch
for sc in 0 1 2 4 6; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras --parity-units 0 --schedule $sc > gpurun_out/sch/b$sc.log 2>&1
python -c "
import json
for l in open('gpurun_out/sch/b$sc.log'):
    if l.startswith('{'):
        d=json.loads(l); print('schedule $sc attend', d['value'])
" || tail -2 gpurun_out/sch/b$sc.log
done
