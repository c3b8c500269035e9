"""Host cost of publishing a drafter snapshot (apply_grad: arena allocation + copy + SGD) and of
freeing one, at the 3B EAGLE drafter. Usage: python tools/snapshot_cost.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2510_26475_b200 as rb  # noqa: E402

shape = rb.TransformerShape.qwen2_5_3b(max_ctx=2048)
tgt = rb.TransformerModel(shape, seed=1)
drf = rb.EagleDrafter(tgt, seed=2, version=1)
grad = drf.new_grad()
torch.cuda.synchronize()
for it in range(5):
    t0 = time.perf_counter()
    new = drf.apply_grad(grad, -0.5)
    t1 = time.perf_counter()
    del new  # refcount drop: rs_model_release -> ~DrafterModel
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"it {it}: apply_grad {1e3 * (t1 - t0):.2f} ms, free {1e3 * (t2 - t1):.2f} ms", flush=True)
# three live snapshots, then released: two are parked (pool size 2), the third is cudaFree'd
snaps = [drf.apply_grad(grad, -0.5) for _ in range(3)]
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    snaps.pop()
    torch.cuda.synchronize()
    print(f"release {i}: {1e3 * (time.perf_counter() - t0):.2f} ms ({'parked' if i < 2 else 'cudaFree'})", flush=True)
