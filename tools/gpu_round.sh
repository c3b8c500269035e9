#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list and one ncu --set full capture.
# usage: gpurun -- bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; cat $O/bench.json
timeout 300 python tools/gemm_cublas_bench.py 1344 > $O/gemm_cublas.log 2>&1; echo "cublas rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "draft/" --nvtx-include "verify/" --nvtx-include "accept/" \
  --csv --log-file $O/launches.csv python tools/profile_step.py 3 > $O/launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:gemm -s 0 -c 4 \
  -o $O/gemm_full python tools/profile_step.py 2 > $O/gemm_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:gemm -s 144 -c 2 \
  -o $O/lmhead_full python tools/profile_step.py 2 > $O/lmhead_full.log 2>&1; echo "ncu lmhead rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "accept/" -k regex:"accept|compact" -s 0 -c 4 \
  -o $O/accept_full python tools/profile_step.py 2 > $O/accept_full.log 2>&1; echo "ncu accept rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:attn_tc -s 2 -c 1 \
  -o $O/attn_full python tools/profile_step.py 2 > $O/attn_full.log 2>&1; echo "ncu attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "verify/" -k regex:gemm -s 0 -c 4 \
  -o $O/gemm_b256_full python tools/profile_step.py 1 1664 256 > $O/gemm_b256_full.log 2>&1; echo "ncu gemm b256 rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx \
  --nvtx-include "verify/" -k regex:gemm --csv --log-file $O/gemm_traffic.csv python tools/profile_step.py 1 > $O/gemm_traffic.log 2>&1
echo "ncu traffic rc=$?"
python tools/gemm_traffic.py $O/gemm_traffic.csv > $O/gemm_traffic.json; head -3 $O/gemm_traffic.json
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --nvtx \
  --nvtx-include "accept/" -k regex:"accept|compact" --csv --log-file $O/accept_traffic.csv python tools/profile_step.py 1 > $O/accept_traffic.log 2>&1
python tools/gemm_traffic.py $O/accept_traffic.csv accept > $O/accept_traffic.json; head -3 $O/accept_traffic.json
python tools/gemm_traffic.py $O/accept_traffic.csv compact > $O/compact_traffic.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kd_elem|kd_lse|kd_tile_stats|row_stats" -s 0 -c 4 \
  -o $O/kd_full python tools/profile_kd.py 1 1664 65 > $O/kd_full.log 2>&1; echo "ncu kd rc=$?"
python tools/ncu_summary.py $O > $O/ncu_summary.md 2> $O/ncu_summary.err; echo "summary rc=$?"
# keep the copy-back under gpurun's 64 MiB: summaries stay, the large reports go
find $O -name "*.ncu-rep" -size +6M -delete
ls -la $O
