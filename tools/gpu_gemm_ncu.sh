#!/bin/bash
# ncu --set full of the first verify GEMMs (QKV+RoPE, O, gate/up, down of layer 0) with source lines
TAG=${1:-gemm_ncu}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:gemm2 -s 0 -c 4 \
  -o $O/gemm_full python tools/profile_step.py 2 > $O/gemm_full.log 2>&1; echo "ncu rc=$?"
for k in "gemm2_kernel<192, 5>" "gemm2_kernel<160, 2>"; do echo "== $k"; python tools/ncu_hot_lines.py $O/gemm_full.ncu-rep "$k" 25; done > $O/hot_lines.txt 2>&1
cat $O/hot_lines.txt | head -70
