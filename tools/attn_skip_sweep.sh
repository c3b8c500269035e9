#!/bin/bash
# attention cost decomposition (RS_TUNE attn_skip bits; results are wrong by design)
for s in ${SKIPS:-0 6 14 22 30 7}; do echo "14b skip=$s"; RS_TUNE=attn_skip=$s timeout 120 python tools/attn_bench.py 32 8192 2 14b 2>&1 | grep verify; done
for s in ${SKIPS3:-0 6 14 22 7}; do echo "3b skip=$s"; RS_TUNE=attn_skip=$s timeout 120 python tools/attn_bench.py 64 1664 2 3b 2>&1 | grep verify; done
