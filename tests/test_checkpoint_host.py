"""CPU: checkpoint naming of the Python mirror (HF Qwen2 / EAGLE-3 names -> C-ABI tensor names)."""
import paper_2510_26475_b200 as rb


def test_checkpoint_names_split():
    t = rb.TransformerModel.__new__(rb.TransformerModel)
    t.shape = rb.TransformerShape.qwen2_5_3b()
    names = t.checkpoint_names()
    assert len(names) == 2 + 36 * 12
    assert t._split("model.layers.7.self_attn.q_proj.weight") == ("q_proj.weight", 7)
    assert t._split("model.layers.35.mlp.down_proj.weight") == ("down_proj.weight", 35)
    assert t._split("model.layers.0.input_layernorm.weight") == ("input_layernorm.weight", 0)
    assert t._split("model.embed_tokens.weight") == ("embed_tokens.weight", -1)
    assert t._split("model.norm.weight") == ("norm.weight", -1)
    d = rb.EagleDrafter.__new__(rb.EagleDrafter)
    dn = d.checkpoint_names()
    assert "midlayer.hidden_norm.weight" in dn and "fc.weight" in dn and len(dn) == 16
    assert d._split("midlayer.input_layernorm.weight") == ("input_layernorm.weight", 0)
    assert d._split("midlayer.mlp.gate_proj.weight") == ("gate_proj.weight", 0)
    t.handle = d.handle = None  # no library handle to release
