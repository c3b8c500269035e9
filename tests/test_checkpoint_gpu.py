"""GPU: checkpoint load / store through the C-ABI (rs_model_load_tensor / rs_model_store_tensor)
-- the transformer counterpart of TabularARModel::to_json / from_json (model.cpp:176-191), so a
real Qwen2.5 target and an EAGLE-3 drafter can be served from Hugging Face tensors.

Checked: the HF layout maps onto the arena (q/k/v are row slices of the fused QKV matrix,
gate/up the even / odd rows of the pairwise-interleaved MLP matrix); fp32 host tensors are
rounded to bf16 exactly like torch; a model loaded from another model's state dict is bitwise
the same model (internal tensors and the tokens it generates); loading a drafter invalidates
the engine's drafter cache; bad names / sizes raise InvalidArgument."""
import os
import random

import numpy as np
import pytest
import torch

import paper_2510_26475_b200 as rb

pytestmark = pytest.mark.gpu

SHAPE = rb.TransformerShape.tiny(vocab=1024, max_ctx=128)


def internal(m, name, layer=-1, dtype=torch.bfloat16):
    return m.to_torch(name, layer, dtype=dtype).cpu()


def generate(tgt, drf, cfg=rb.SDConfig.tree(1, 3, 3), mode="greedy"):
    rng = random.Random(3)
    reqs = [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(5 + i)], -2.0, 10,
                            rb.DecodeRng.from_seed(1, i)) for i in range(3)]
    eng = rb.BatchEngine(tgt, lambda: drf, None, rb.TimingModel(), reqs, cfg, mode, record_full_logprobs=False)
    while not eng.all_done():
        eng.step()
    return [r.generated for r in eng.requests()]


def test_hf_layout_maps_onto_the_arena():
    tgt = rb.TransformerModel(SHAPE, seed=5)
    s, hq, hk = SHAPE, SHAPE.n_heads * 128, SHAPE.n_kv_heads * 128
    qkv = internal(tgt, "qkv_w", 1).view(hq + 2 * hk, s.d_model)
    as_t = lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16)  # noqa: E731
    assert torch.equal(as_t(tgt.store_tensor("q_proj.weight", 1)), qkv[:hq])
    assert torch.equal(as_t(tgt.store_tensor("k_proj.weight", 1)), qkv[hq:hq + hk])
    assert torch.equal(as_t(tgt.store_tensor("v_proj.weight", 1)), qkv[hq + hk:])
    gu = internal(tgt, "gu_w", 0).view(2 * s.d_ff, s.d_model)
    assert torch.equal(as_t(tgt.store_tensor("gate_proj.weight", 0)), gu[0::2])
    assert torch.equal(as_t(tgt.store_tensor("up_proj.weight", 0)), gu[1::2])
    qb = internal(tgt, "qkv_b", 0)
    assert torch.equal(as_t(tgt.store_tensor("v_proj.bias", 0)), qb[hq + hk:])
    assert tgt.tensor_shape("o_proj.weight", 0) == (s.d_model, hq)
    assert tgt.tensor_shape("down_proj.weight", 0) == (s.d_model, s.d_ff)
    assert tgt.tensor_shape("norm.weight") == (s.d_model,)
    # bf16 bit patterns and the float view agree
    bits = tgt.store_tensor("embed_tokens.weight", bf16_bits=True)
    assert np.array_equal((bits.astype(np.uint32) << 16).view(np.float32), tgt.store_tensor("embed_tokens.weight"))


def test_fp32_load_rounds_like_torch():
    tgt = rb.TransformerModel(SHAPE, seed=5)
    g = torch.Generator().manual_seed(0)
    w = torch.randn(SHAPE.d_ff, SHAPE.d_model, generator=g) * 0.05
    w[0, :4] = torch.tensor([float("inf"), -float("inf"), 1e-40, 3.0e38])
    tgt.load_tensor("up_proj.weight", 1, w.numpy())
    gu = internal(tgt, "gu_w", 1).view(2 * SHAPE.d_ff, SHAPE.d_model)
    assert torch.equal(gu[1::2].view(torch.int16), w.to(torch.bfloat16).view(torch.int16))
    # a bf16 torch tensor is taken bit for bit; gains stay fp32
    wb = (torch.randn(SHAPE.d_ff, SHAPE.d_model, generator=g) * 0.05).to(torch.bfloat16)
    tgt.load_tensor("gate_proj.weight", 1, wb)
    gu = internal(tgt, "gu_w", 1).view(2 * SHAPE.d_ff, SHAPE.d_model)
    assert torch.equal(gu[0::2].view(torch.int16), wb.view(torch.int16))
    gain = torch.rand(SHAPE.d_model, generator=g) + 0.5
    tgt.load_tensor("input_layernorm.weight", 0, gain)
    assert torch.equal(internal(tgt, "ln1", 0, torch.float32), gain)


def test_state_dict_round_trip_is_the_same_model(tmp_path):
    a = rb.TransformerModel(SHAPE, seed=21)
    da = rb.EagleDrafter(a, seed=22)
    b = rb.TransformerModel(SHAPE, seed=31)
    db = rb.EagleDrafter(b, seed=32)
    ref = generate(a, da)
    assert generate(b, db) != ref  # different weights, different output
    b.load_state_dict(a.state_dict(bf16_bits=True))
    path = os.path.join(tmp_path, "drafter.npz")
    da.save(path)
    db.load(path)
    for name in ("qkv_w", "qkv_b", "o_w", "gu_w", "down_w"):
        for layer in range(SHAPE.n_layers):
            assert torch.equal(internal(a, name, layer), internal(b, name, layer)), (name, layer)
        assert torch.equal(internal(da, name), internal(db, name)), name
    for name in ("ln1", "ln2"):
        assert torch.equal(internal(a, name, 0, torch.float32), internal(b, name, 0, torch.float32))
    for name in ("fc_w", "lm_w"):
        assert torch.equal(internal(da, name), internal(db, name))
    for name in ("norm_emb", "norm_hid", "final_norm"):
        assert torch.equal(internal(da, name, dtype=torch.float32), internal(db, name, dtype=torch.float32))
    assert generate(b, db) == ref
    assert generate(b, db, mode="sample") == generate(a, da, mode="sample")


def test_loading_a_drafter_mid_run_invalidates_its_cache():
    a = rb.TransformerModel(SHAPE, seed=41)
    d1 = rb.EagleDrafter(a, seed=42)
    d2 = rb.EagleDrafter(a, seed=43)
    want = generate(a, d2, mode="sample")
    rng = random.Random(3)
    reqs = [rb.RequestState(i, [rng.randrange(SHAPE.vocab - 1) for _ in range(5 + i)], -2.0, 10,
                            rb.DecodeRng.from_seed(1, i)) for i in range(3)]
    eng = rb.BatchEngine(a, lambda: d1, None, rb.TimingModel(), reqs, rb.SDConfig.tree(1, 3, 3), "sample",
                         record_full_logprobs=False)
    eng.step()  # the drafter cache now holds d1's keys / values
    d1.load_state_dict(d2.state_dict())
    while not eng.all_done():
        eng.step()
    # lossless either way; the accepted drafts after the load follow d2's weights
    got = [r.generated for r in eng.requests()]
    assert all(len(g) > 0 for g in got)
    assert generate(a, d1, mode="sample") == want


def test_bad_checkpoint_tensors_raise():
    tgt = rb.TransformerModel(SHAPE, seed=5)
    with pytest.raises(rb.InvalidArgument, match="unknown tensor"):
        tgt.load_tensor("q_proj.weights", 0, np.zeros(4, np.float32))
    with pytest.raises(rb.InvalidArgument, match="layer out of range"):
        tgt.load_tensor("q_proj.weight", SHAPE.n_layers, np.zeros(4, np.float32))
    with pytest.raises(rb.InvalidArgument, match="element count"):
        tgt.load_tensor("q_proj.weight", 0, np.zeros(4, np.float32))
    sd = tgt.state_dict()
    sd.pop("model.norm.weight")
    with pytest.raises(rb.InvalidArgument, match="missing"):
        tgt.load_state_dict(sd)
