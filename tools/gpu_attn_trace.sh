#!/bin/bash
# attention per-pass trace + per-CTA timeline at cfg2 geometry (layer 1) under variants
TAG=${1:-attn_trace}
O=gpurun_out/$TAG
mkdir -p $O
for cfg in ${CFGS:-attn_skip=0}; do
  RS_TUNE=attn_trace=2,$cfg timeout 120 python tools/attn_bench.py 64 1664 2 3b 2>&1 | grep -v " -1 " > $O/trace_$cfg.log; echo "$cfg rc=$?"; grep CTAs $O/trace_$cfg.log | tail -3
done
