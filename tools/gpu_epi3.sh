#!/bin/bash
# third epilogue group on single-wave SM-pair GEMMs: GEMM / engine parity, then a same-process A/B
TAG=${1:-epi3}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or qkv or parity_qwen or tree_attn" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python tools/ab_step.py epi3 0 -1 6 8 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -4 $O/ab.log
RS_TUNE=gemm_trace=1 timeout 300 python tools/profile_step.py 1 > $O/trace.log 2>&1; grep "gemm2 F=" $O/trace.log | head -12
