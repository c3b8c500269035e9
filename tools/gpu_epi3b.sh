#!/bin/bash
# third epilogue group: whole GPU suite + bench, a longer same-process A/B and the verify GEMM trace
TAG=${1:-epi3b}
O=gpurun_out/$TAG
bash tools/gpu_full.sh $TAG
timeout 600 python tools/ab_step.py epi3 0 -1 10 8 > $O/ab.log 2>&1; echo "ab rc=$?"; tail -2 $O/ab.log
for f in 0 -1; do
  RS_TUNE=gemm_trace=1,epi3=$f timeout 300 python tools/profile_step.py 2 > $O/trace_$f.log 2>&1
  echo "epi3=$f"; grep "gemm2 F=" $O/trace_$f.log | grep "T=1344" | tail -3
done
