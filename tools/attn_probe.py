"""Probe the target attention kernel on a few shapes (each case in a subprocess with a timeout)."""
import subprocess
import sys
import os

CASE = r'''
import random, sys
sys.path.insert(0, "{root}")
import paper_2510_26475_b200 as rb
H, KV, plen, L, cfg = {H}, {KV}, {plen}, {L}, rb.SDConfig.tree(1, 4, 5)
shape = rb.TransformerShape(1024, 256, L, H, KV, 128, 512, 1024)
tgt = rb.TransformerModel(shape, seed=3)
drf = rb.EagleDrafter(tgt, seed=4)
print("created", flush=True)
rng = random.Random(0)
reqs = [rb.RequestState(i, [rng.randrange(1023) for _ in range(plen)], -2.0, 8, rb.DecodeRng.from_seed(1, i)) for i in range({B})]
eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, cfg, "greedy", record_full_logprobs=False)
print("prefilled", flush=True)
k = 0
while not eng.all_done() and k < 4:
    eng.step(); k += 1
print("stepped", k, flush=True)
'''

cases = [dict(H=4, KV=2, plen=20, L=1, B=2), dict(H=4, KV=2, plen=300, L=1, B=2),
         dict(H=16, KV=2, plen=20, L=1, B=2), dict(H=16, KV=2, plen=100, L=1, B=2),
         dict(H=16, KV=2, plen=300, L=1, B=2), dict(H=16, KV=2, plen=300, L=2, B=4)]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for c in cases:
    code = CASE.format(root=root, **c)
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=float(os.environ.get("T", 60)))
        print(c, "rc", r.returncode, r.stdout.strip().replace("\n", " | "), r.stderr.strip()[-300:])
    except subprocess.TimeoutExpired as e:
        print(c, "TIMEOUT", (e.stdout or b"").decode() if isinstance(e.stdout, bytes) else e.stdout)
    sys.stdout.flush()
