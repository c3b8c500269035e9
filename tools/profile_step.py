"""Run the cfg2 engine for a few steps (for ncu captures). Usage: python tools/profile_step.py [steps] [ctx] [batch]"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1664
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 64
shape = rb.TransformerShape.qwen2_5_3b(max_ctx=ctx + 256)
tgt = rb.TransformerModel(shape, seed=20251026)
drf = rb.EagleDrafter(tgt, seed=4242, version=1)
rng = random.Random(1000)
reqs = [rb.RequestState(i, [rng.randrange(shape.vocab - 1) for _ in range(ctx)], -20.0, 200,
                        rb.DecodeRng.from_seed(7, i)) for i in range(batch)]
eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 4, 5), "sample",
                     record_full_logprobs=False)
print("prefill launches", rb.launch_count(), flush=True)
for _ in range(steps):
    info = eng.step()
    print("step", info.step_ms, info.emitted_tokens, rb.launch_count(), flush=True)
