#!/bin/bash
# Attention diagnosis: per-pass trace of CTA 0 (cfg2 geometry) and the skip decomposition.
TAG=${1:-attn_diag}
O=gpurun_out/$TAG
mkdir -p $O
RS_TUNE=attn_trace=2 timeout 300 python tools/attn_bench.py 64 1664 2 3b > $O/trace_3b.log 2>&1; echo "trace rc=$?"
SKIPS3="0 1 2 4 6 3 5 7" SKIPS="0 1 6 7" bash tools/attn_skip_sweep.sh > $O/skip.log 2>&1; echo "skip rc=$?"; cat $O/skip.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 1500 $O/bench.json
