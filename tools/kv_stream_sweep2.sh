#!/bin/bash
B=tools/kv_stream_bench
for it in 128 148; do for d in "2 2" "4 4" "6 6" "7 6"; do $B $it 8256 $d 0; done; done
for d in "2 2" "4 4" "7 6"; do $B 128 1728 $d 0 1000; done
for pf in 4 8 16 32; do $B 128 1728 4 4 4 0 $pf; $B 128 1728 4 4 4 1000 $pf; $B 128 1728 2 2 4 1500 $pf; done
for pf in 8 16 32; do $B 256 8256 4 4 4 1500 $pf; done
