#!/bin/bash
# compute-sanitizer on the final epilogue changes (third epilogue group, relaxed arrive, shared-space staging)
TAG=${1:-sanitize2}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q > $O/gemm_tests.log 2>&1; echo "gemm tests rc=$?"; tail -2 $O/gemm_tests.log
timeout 1500 compute-sanitizer --tool racecheck python -m pytest tests/test_gemm_gpu.py -x -q -k "third_epilogue and (256-2048-4096 or 300-2048-2048)" > $O/racecheck_gemm.log 2>&1; echo "racecheck gemm rc=$?"; grep -c "Race reported" $O/racecheck_gemm.log; tail -3 $O/racecheck_gemm.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gemm_gpu.py -x -q -k "third_epilogue and (256-2048-4096 or 300-2048-2048)" > $O/memcheck_gemm.log 2>&1; echo "memcheck gemm rc=$?"; tail -3 $O/memcheck_gemm.log
bash tools/gpu_sanitize.sh $TAG
