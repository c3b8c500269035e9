"""GPU: the CPU transformer port (oracle/tf_cpu.cpp) generates the SAME synthetic weights as the
CUDA models (model.cu init_normal_kernel: splitmix64 -> Box-Muller -> bf16, same tensor ids), so
the bench's same-workload CPU timing (cpu_baseline.same_workload_port) runs exactly the models the
GPU serves; and its rows match the CUDA engine's captured rows within the logits bar."""
import random

import numpy as np
import pytest
import torch

import paper_2510_26475_b200 as rb
from oracle_client import Oracle

pytestmark = pytest.mark.gpu

SHAPE = rb.TransformerShape.tiny(vocab=1024, max_ctx=128)
JS = {"V": SHAPE.vocab, "d": SHAPE.d_model, "L": SHAPE.n_layers, "H": SHAPE.n_heads, "KV": SHAPE.n_kv_heads,
      "dff": SHAPE.d_ff}


@pytest.fixture(scope="module")
def both():
    orc = Oracle()
    pid = orc("tf_cpu_create", shape=JS, seed=11, drafter_seed=12)["id"]
    tgt = rb.TransformerModel(SHAPE, seed=11)
    drf = rb.EagleDrafter(tgt, seed=12)
    yield orc, pid, tgt, drf
    orc("tf_cpu_free", id=pid)


def bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def test_same_synthetic_weights(both):
    orc, pid, tgt, drf = both
    for name, layer, m, dr in (("emb", -1, tgt, False), ("qkv_w", 0, tgt, False), ("gu_w", 1, tgt, False),
                               ("down_w", 1, tgt, False), ("qkv_b", 1, tgt, False), ("fc_w", -1, drf, True),
                               ("lm_w", -1, drf, True), ("o_w", -1, drf, True)):
        port = np.array(orc("tf_cpu_tensor", id=pid, name=name, layer=max(layer, 0), drafter=dr)["bits"], np.uint16)
        assert np.array_equal(port, bits(m.to_torch(name, layer))), name


def test_port_rows_match_the_cuda_engine(both):
    orc, pid, tgt, drf = both
    rng = random.Random(2)
    reqs = [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(8 + i)], -2.0, 8,
                            rb.DecodeRng.from_seed(3, i)) for i in range(2)]
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 2, 3), "sample",
                         record_full_logprobs=False)
    eng.set_capture(True)
    while not eng.all_done():
        eng.step()
    done = eng.requests()
    full = [r.prompt + r.generated for r in done]
    worst, checked = 0.0, 0
    for role, req, cl, ext, logits in eng.captured_rows():
        ctx = full[req][:cl] + ext
        args = dict(role="drafter", depth=len(ext)) if role == 0 else {}
        got = torch.tensor(orc("tf_cpu_logits", id=pid, ctx=ctx, **args)["logits"])
        ref = torch.tensor(logits, dtype=torch.float32)
        worst = max(worst, (got - ref).abs().max().item() / ref.std().item())
        checked += 1
        if checked >= 40:
            break
    assert checked >= 10 and worst < 3e-2, worst
