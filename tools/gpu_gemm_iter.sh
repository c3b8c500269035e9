#!/bin/bash
# GEMM iteration: GEMM + transformer parity tests, one-step GEMM timeline, short bench
TAG=${1:-gemm_iter}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_transformer_gpu.py tests/test_parity_qwen_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
RS_TUNE=gemm_trace=1 timeout 300 python tools/profile_step.py 2 > $O/trace.log 2>&1; grep "gemm2 F" $O/trace.log | tail -6
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg > $O/bench$r.json 2> $O/bench$r.err
python -c "
import json; d=json.load(open('$O/bench$r.json'))
print(d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['breakdown_ms_per_step']['verify.gemm'])
"
done
