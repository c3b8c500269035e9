#!/bin/bash
# lazy verify LM head: the parity suites that run the SD engine, then the bench with it on / off
TAG=${1:-lazy}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for f in 0 -1; do
  RS_TUNE=lazy_lm=$f timeout 600 python bench.py --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg > $O/bench_$f.json 2> $O/bench_$f.err
  python -c "
import json; d=json.load(open('$O/bench_$f.json'))
print('lazy $f', d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['parity']['greedy_sd_equals_greedy_decode'])
for k,v in list(d['breakdown_ms_per_step'].items())[:5]: print('  ', k, v)
"
done
