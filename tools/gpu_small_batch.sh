#!/bin/bash
# launch-overhead check at the tuner's small buckets: device-timed vs end-to-end tokens/s
TAG=${1:-small}
O=gpurun_out/$TAG
mkdir -p $O
for b in 1 4 16; do
  timeout 300 python bench.py --batch $b --steps 20 --warmup 5 --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg --no-profile > $O/b$b.json 2> $O/b$b.err
  python -c "
import json; d=json.load(open('$O/b$b.json'))
print('batch $b', 'device', d['value'], 'e2e', d['e2e']['value'], 'ms/step', d['ms_per_step'], 'launches', d['gpu_launches'])
"
done
