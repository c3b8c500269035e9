#!/bin/bash
# acceptance register-budget variants: parity (cluster / replay tests) and the bench's acceptance time
TAG=${1:-acc_iter}
O=gpurun_out/$TAG
mkdir -p $O
for mb in 4 3; do
  RS_TUNE=accept_minb=$mb timeout 900 python -m pytest tests/test_accept_cluster_gpu.py tests/test_parity_qwen_gpu.py -x -q -k "cluster or replay" > $O/pytest_$mb.log 2>&1; echo "pytest mb=$mb rc=$?"; tail -1 $O/pytest_$mb.log
done
for mb in 1 4 3; do
  RS_TUNE=accept_minb=$mb timeout 600 python bench.py --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg > $O/bench_$mb.json 2> $O/bench_$mb.err
  python -c "
import json; d=json.load(open('$O/bench_$mb.json'))
print('mb $mb', d['ms_per_step'], d['clocks']['sm_mhz'], d['breakdown_ms_per_step']['accept.accept'])
"
done
