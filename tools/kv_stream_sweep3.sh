#!/bin/bash
B=tools/kv_stream_bench
for h in 0 5 6 7; do $B 128 1728 5 4 0 0 8 $h; done
for h in 0 5 6; do $B 256 8256 5 4 0 0 8 $h; done
