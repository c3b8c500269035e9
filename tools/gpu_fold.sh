#!/bin/bash
# folded RMSNorm: parity tests that run the target forward, then the bench with the fold on / off
TAG=${1:-fold}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_transformer_gpu.py tests/test_parity_qwen_gpu.py tests/test_gemm_gpu.py tests/test_kd_transformer_gpu.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
grep -E "cuda vs fp32" $O/pytest.log | head
for f in 0 -1; do
  RS_TUNE=fold_norm=$f timeout 600 python bench.py --no-cpu-baseline --kd 0 --no-tuner-leg --no-b256-leg > $O/bench_$f.json 2> $O/bench_$f.err
  python -c "
import json; d=json.load(open('$O/bench_$f.json'))
print('fold $f', d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['parity'])
for k,v in list(d['breakdown_ms_per_step'].items())[:6]: print('  ', k, v)
"
done
