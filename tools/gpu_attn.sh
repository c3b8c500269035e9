#!/bin/bash
# Attention iteration: the micro-bench at cfg2 / batch-256 / 14B-8K geometry (first, under short
# timeouts, so a hang costs minutes), the parity tests that exercise the tensor-core attention,
# and a per-pass trace + per-CTA timeline.
TAG=${1:-attn}
O=gpurun_out/$TAG
mkdir -p $O
timeout 150 python tools/attn_bench.py 64 1664 2 3b > $O/attn_3b.log 2>&1; rc=$?; echo "attn3b rc=$rc"; tail -2 $O/attn_3b.log
if [ $rc -ne 0 ]; then exit 1; fi
for p in ${POLYS:-1 2}; do RS_TUNE=attn_poly=$p timeout 150 python tools/attn_bench.py 64 1664 2 3b > $O/attn_3b_poly$p.log 2>&1; echo "attn3b poly$p rc=$?"; tail -1 $O/attn_3b_poly$p.log; done
timeout 150 python tools/attn_bench.py 256 1664 2 3b > $O/attn_3b_b256.log 2>&1; echo "attn3b256 rc=$?"; tail -1 $O/attn_3b_b256.log
timeout 150 python tools/attn_bench.py 32 8192 2 14b > $O/attn_14b.log 2>&1; echo "attn14b rc=$?"; tail -1 $O/attn_14b.log
for p in ${POLYS:-1 2}; do RS_TUNE=attn_poly=$p timeout 150 python tools/attn_bench.py 32 8192 2 14b > $O/attn_14b_poly$p.log 2>&1; echo "attn14b poly$p rc=$?"; tail -1 $O/attn_14b_poly$p.log; done
timeout 900 python -m pytest tests/test_transformer_gpu.py tests/test_parity_qwen_gpu.py tests/test_accept_cluster_gpu.py ${EXTRA_TESTS} -x -q > $O/pytest_attn.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_attn.log
RS_TUNE=attn_trace=2 timeout 120 python tools/attn_bench.py 64 1664 2 3b 2>&1 | grep -v " -1 " > $O/trace_3b.log; echo "trace rc=$?"; grep CTAs $O/trace_3b.log | tail -1
