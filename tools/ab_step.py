"""A/B of one tuning key on the cfg2 engine step in ONE process (same clocks): alternating blocks of
timed steps with the key at each value. Usage: python tools/ab_step.py key valueA valueB [blocks] [steps]"""
import os
import random
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

key, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
blocks = int(sys.argv[4]) if len(sys.argv) > 4 else 4
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 8
ctx, batch = 1664, 64
max_len = blocks * 2 * (steps + 1) * 6 + 32
shape = rb.TransformerShape.qwen2_5_3b(max_ctx=ctx + max_len + 64)
tgt = rb.TransformerModel(shape, seed=20251026)
drf = rb.EagleDrafter(tgt, seed=4242, version=1)
rng = random.Random(1000)
reqs = [rb.RequestState(i, [rng.randrange(shape.vocab - 1) for _ in range(ctx)], -20.0, max_len,
                        rb.DecodeRng.from_seed(7, i)) for i in range(batch)]
dev = rb.default_device()
s = torch.cuda.Stream()
dev.set_stream(s.cuda_stream)
eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 4, 5), "sample",
                     record_full_logprobs=False, device=dev)
for _ in range(3):
    eng.step()
res = {va: [], vb: []}
for b in range(blocks):
    for v in ((va, vb) if b % 2 == 0 else (vb, va)):
        rb.set_tuning(key, v)
        eng.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            eng.step()
        e1.record(s)
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / steps)
for v in (va, vb):
    print(f"{key}={v}: ms/step {sorted(round(x, 3) for x in res[v])} mean {sum(res[v]) / len(res[v]):.3f}")
