#!/bin/bash
# compute-sanitizer over the smoke and the round-2 test additions (tiny shapes; memcheck + racecheck on smoke)
TAG=${1:-sanitize}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -2 $O/memcheck_smoke.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_checkpoint_gpu.py tests/test_tf_cpu_gpu.py tests/test_transformer_gpu.py tests/test_kd_transformer_gpu.py -x -q > $O/memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -3 $O/memcheck_tests.log
timeout 1800 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > $O/racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"; grep -c "Race reported" $O/racecheck_smoke.log; grep "Race reported" $O/racecheck_smoke.log | sed 's/0x[0-9a-f]*//g' | sort | uniq -c | head; tail -2 $O/racecheck_smoke.log
