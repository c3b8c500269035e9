#!/bin/bash
# Attention iteration: parity tests that exercise the tensor-core attention, the micro-bench at
# cfg2 / 14B-8K geometry, and a GEMM timeline trace of one step.
TAG=${1:-attn}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_transformer_gpu.py tests/test_parity_qwen_gpu.py tests/test_accept_cluster_gpu.py -x -q > $O/pytest_attn.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_attn.log
timeout 300 python tools/attn_bench.py 64 1664 2 3b > $O/attn_3b.log 2>&1; echo "attn3b rc=$?"; cat $O/attn_3b.log | tail -4
timeout 300 python tools/attn_bench.py 256 1664 2 3b > $O/attn_3b_b256.log 2>&1; echo "attn3b256 rc=$?"; cat $O/attn_3b_b256.log | tail -4
timeout 300 python tools/attn_bench.py 32 8192 2 14b > $O/attn_14b.log 2>&1; echo "attn14b rc=$?"; cat $O/attn_14b.log | tail -4
RS_TUNE=gemm_trace=1 timeout 300 python tools/profile_step.py 2 > $O/gemm_trace.log 2>&1; echo "trace rc=$?"
