"""Target-attention timing at the bench's geometry without the whole model: a Qwen2.5-3B-headed
target with few layers (attention cost per layer does not depend on depth), batch 64, context
1664, tree(1,4,5); per-layer verify attention time from the device profiler.

    python tools/attn_bench.py [batch] [ctx] [layers] [model]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1664
L = int(sys.argv[3]) if len(sys.argv) > 3 else 2
model = sys.argv[4] if len(sys.argv) > 4 else "3b"
geo = {"3b": (151936, 2048, 16, 2, 11008), "7b": (152064, 3584, 28, 4, 18944), "14b": (152064, 5120, 40, 8, 13824)}[model]
V, d, H, KV, dff = geo
shape = rb.TransformerShape(V, d, L, H, KV, 128, dff, max_ctx=ctx + 256)
tgt = rb.TransformerModel(shape, seed=1)
drf = rb.EagleDrafter(tgt, seed=2)
rng = random.Random(0)
reqs = [rb.RequestState(i, [rng.randrange(V - 1) for _ in range(ctx)], -20.0, 200, rb.DecodeRng.from_seed(1, i))
        for i in range(B)]
eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 4, 5), "sample",
                     record_full_logprobs=False)
for _ in range(3):
    eng.step()
rb.device_profile(enable=True, reset=True)
n = 5
for _ in range(n):
    eng.step()
prof = rb.device_profile(enable=False)
for k in sorted(prof):
    if "attn" in k:
        v = prof[k]
        per = v["ms"] / v["launches"] * 1e3
        gbs = v["bytes"] / (v["ms"] / 1e3) / 1e9
        print(f"{k:16s} launches {v['launches']:4d}  {per:8.2f} us/launch  {gbs:8.1f} GB/s (algorithmic K/V bytes)")
