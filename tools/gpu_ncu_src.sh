#!/bin/bash
# ncu --set full with SASS source of layer 0's verify QKV / O GEMMs and one target attention launch
TAG=${1:-ncusrc}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:gemm2 -s 0 -c 4 \
  -o $O/gemm python tools/profile_step.py 2 > $O/gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:attn_tc -s 2 -c 1 \
  -o $O/attn python tools/profile_step.py 2 > $O/attn.log 2>&1; echo "ncu attn rc=$?"
for i in 0 1 2 3; do ncu -i $O/gemm.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > $O/gemm_src_$i.csv 2>&1; done
ncu -i $O/attn.ncu-rep --page source --csv --print-source sass > $O/attn_src.csv 2>&1
ncu -i $O/gemm.ncu-rep --page details --csv > $O/gemm_details.csv 2>&1
ncu -i $O/attn.ncu-rep --page details --csv > $O/attn_details.csv 2>&1
find $O -name "*.ncu-rep" -size +20M -delete
ls -la $O
