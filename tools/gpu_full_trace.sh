#!/bin/bash
# gpu_full.sh plus the verify GEMM timeline trace (RS_TUNE=gemm_trace=1) and a same-process A/B of the epi3 key
TAG=${1:-fulltrace}
O=gpurun_out/$TAG
bash tools/gpu_full.sh $TAG
RS_TUNE=gemm_trace=1 timeout 300 python tools/profile_step.py 2 > $O/trace.log 2>&1
grep "gemm2 F=" $O/trace.log | grep "T=1344" > $O/trace_verify.log
python - <<PY
import re,statistics as st
d={}
for l in open('$O/trace_verify.log'):
    m=re.search(r"F=(\d+) T=1344 K=(\d+) BT=(\d+) epi=(\d+): wait (\d+) full0 (\d+) mma_done (\d+) epi (\d+)\.\.(\d+) exit (\d+)",l)
    if not m: continue
    F,K,BT,E,w,f0,md,e0,e1,ex=map(int,m.groups())
    d.setdefault((F,K,BT,E),[]).append((e1-e0, ex-md, ex))
for k,v in sorted(d.items()):
    print(k,len(v),'epi',st.median([a for a,b,c in v]),'mma_done->exit',st.median([b for a,b,c in v]),'exit',st.median([c for a,b,c in v]))
PY
timeout 600 python tools/ab_step.py epi3 0 -1 6 8 > $O/ab.log 2>&1; tail -2 $O/ab.log
