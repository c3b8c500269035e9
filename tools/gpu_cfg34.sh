#!/bin/bash
# BASELINE cfg3 (7B, measured tuner) and cfg4 (14B, 8K contexts, rejection sampling T=1) on one GPU
TAG=${1:-cfg34}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 python bench.py --model 7b --batch 32 --tuner --no-cpu-baseline --kd 0 --no-b256-leg > $O/cfg3.json 2> $O/cfg3.err; echo "cfg3 rc=$?"
timeout 1500 python bench.py --model 14b --batch 32 --ctx 8192 --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg > $O/cfg4.json 2> $O/cfg4.err; echo "cfg4 rc=$?"
python -c "
import json
for f in ['cfg3','cfg4']:
    try:
        d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'failed', e)
"
