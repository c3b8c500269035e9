#!/bin/bash
# One default bench run (+ optional GEMM timeline trace of one step)
TAG=${1:-bench}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench.json'))
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks'])
for k,v in list(d['breakdown_ms_per_step'].items())[:6]: print(k, v)
print(json.dumps(d.get('kd_async_overlap')))
"
if [ -n "$TRACE" ]; then RS_TUNE=gemm_trace=1 timeout 300 python tools/profile_step.py 2 > $O/gemm_trace.log 2>&1; echo "trace rc=$?"; grep "gemm2 F" $O/gemm_trace.log | tail -12; fi
