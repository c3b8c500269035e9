#!/bin/bash
# ncu --set full of one acceptance launch (cfg2) with source lines + hot lines
TAG=${1:-accept_ncu}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "accept/" -k regex:accept_kernel -s 1 -c 1 \
  -o $O/accept_full python tools/profile_step.py 3 > $O/accept_full.log 2>&1; echo "ncu rc=$?"
python tools/ncu_hot_lines.py $O/accept_full.ncu-rep accept_kernel 45 > $O/hot_lines.txt 2>&1; cat $O/hot_lines.txt
