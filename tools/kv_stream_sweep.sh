#!/bin/bash
# Sweep of tools/kv_stream_bench (K/V span streaming, no compute) at cfg2 / 14B-8K geometry.
B=tools/kv_stream_bench
for m in 0 1 2 3; do $B 128 1728 5 4 $m; done
for d in "2 2" "4 4" "6 6" "8 5"; do $B 128 1728 $d 0; done
$B 148 1728 5 4 0; $B 256 1728 5 4 0; $B 512 1728 5 4 0
for dl in 500 1000 1500; do $B 128 1728 5 4 0 $dl; done
$B 256 8256 5 4 0; $B 256 8256 5 4 1; $B 256 8256 5 4 3; $B 256 8256 5 4 0 1500
