"""Phase breakdown of one transformer KD update (cfg5 leg). Usage: python tools/profile_kd.py [n] [ctx] [resp]"""
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2510_26475_b200 as rb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 1664
resp = int(sys.argv[3]) if len(sys.argv) > 3 else 65
shape = rb.TransformerShape.qwen2_5_3b(max_ctx=ctx + resp + 64)
tgt = rb.TransformerModel(shape, seed=20251026)
drf = rb.EagleDrafter(tgt, seed=4242, version=1)
rng = random.Random(5)
samples = [rb.RolloutSample([rng.randrange(shape.vocab - 1) for _ in range(ctx)],
                            [rng.randrange(shape.vocab - 1) for _ in range(resp)], [], 0.0, rng.random())
           for _ in range(n)]
w = [1.0] * n
grad = drf.new_grad()
for it in range(3):
    if it == 2:
        rb.device_profile(enable=True, reset=True)
    torch.cuda.synchronize()
    t = time.time()
    loss, _ = rb.kd_grad_transformer(drf, samples, w, grad)
    torch.cuda.synchronize()
    print("kd_grad", it, round((time.time() - t) * 1e3, 2), "ms", loss, flush=True)
prof = rb.device_profile(enable=False)
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:24s} {v['ms']:9.3f} ms  n={v['launches']:5d}  TF/s={v['flops'] / max(v['ms'], 1e-9) / 1e9:8.1f}"
          f"  GB/s={v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
print("total device ms", sum(v["ms"] for v in prof.values()))

# the engine-resident path: generate the responses, then KD from the live engine
reqs = [rb.RequestState(i, list(samples[i].prompt), -20.0, resp, rb.DecodeRng.from_seed(7, i)) for i in range(n)]
eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 4, 5), "sample",
                     record_full_logprobs=False)
while not eng.all_done():
    eng.step()
for it in range(3):
    if it == 2:
        rb.device_profile(enable=True, reset=True)
    torch.cuda.synchronize()
    t = time.time()
    loss, _ = eng.kd_grad(drf, list(range(n)), w, grad)
    t2 = time.time()
    nd = drf.apply_grad(grad, -0.5)
    torch.cuda.synchronize()
    print("apply_grad", round((time.time() - t2) * 1e3, 2), "ms", flush=True)
    torch.cuda.synchronize()
    print("engine kd_grad", it, round((time.time() - t) * 1e3, 2), "ms", loss, flush=True)
prof = rb.device_profile(enable=False)
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{k:24s} {v['ms']:9.3f} ms  n={v['launches']:5d}")
print("total device ms", sum(v["ms"] for v in prof.values()))
