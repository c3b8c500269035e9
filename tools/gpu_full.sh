#!/bin/bash
# Round validation: smoke, the whole GPU test suite, the default bench line.
TAG=${1:-full}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench.json'))
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks'], d['roofline']['frac'])
print(json.dumps(d['cpu_baseline'].get('same_workload_port')))
"
