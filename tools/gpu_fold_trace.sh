#!/bin/bash
TAG=${1:-fold_trace}
O=gpurun_out/$TAG
mkdir -p $O
for f in 0 -1; do
  RS_TUNE=gemm_trace=1,fold_norm=$f timeout 300 python tools/profile_step.py 2 > $O/trace_$f.log 2>&1
  echo "fold $f"; grep "gemm2 F" $O/trace_$f.log | tail -6
done
