#!/bin/bash
# ncu --set full of one verify attention launch at cfg2 geometry (2-layer 3B-headed target)
TAG=${1:-attn_ncu}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:attn_tc -s 3 -c 1 \
  -o $O/attn_full python tools/attn_bench.py 64 1664 2 3b > $O/attn_full.log 2>&1; echo "ncu rc=$?"
python tools/ncu_hot_lines.py $O/attn_full.ncu-rep attn_tc 40 > $O/hot_lines.txt 2>&1; head -50 $O/hot_lines.txt
ncu -i $O/attn_full.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
grep -iE "stall|Duration|Throughput|Pipe|Issue" $O/details.csv | head -80
