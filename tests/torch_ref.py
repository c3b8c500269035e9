"""Plain PyTorch fp32 reference of the transformer forwards (test infrastructure only).

Mirrors the CUDA path's architecture (Qwen2 target, EAGLE-3-style drafter) on the SAME
synthetic weights (copied out of HBM with rs_model_tensor), in fp32 with bf16 rounding at
the points where the CUDA path stores bf16 activations, so the comparison isolates kernel
arithmetic (accumulation order, fast exp) from the model definition.
"""
import torch


def bf(x):
    return x.to(torch.bfloat16).float()


class TargetRef:
    """bf16_mm=True: every matmul takes bf16 operands with fp32 accumulation (cuBLAS bf16
    GEMMs) instead of fp32 -- a second, equally valid bf16 implementation whose distance to
    the fp32 one calibrates the noise floor of the bf16 rounding points."""

    def __init__(self, m, bf16_mm=False):
        s = m.shape
        self.s = s
        self.bf16_mm = bf16_mm
        d, q = s.d_model, (s.n_heads + 2 * s.n_kv_heads) * s.head_dim
        self.emb = m.to_torch("emb").view(s.vocab, d).float()
        self.final = m.to_torch("final_norm").float()
        self.layers = []
        for l in range(s.n_layers):
            gu = m.to_torch("gu_w", l).view(2 * s.d_ff, d).float()  # rows 2i gate_i, 2i+1 up_i
            self.layers.append(dict(
                qkv_w=m.to_torch("qkv_w", l).view(q, d).float(), qkv_b=m.to_torch("qkv_b", l).float(),
                o_w=m.to_torch("o_w", l).view(d, s.n_heads * s.head_dim).float(),
                g_w=gu[0::2], u_w=gu[1::2],
                down_w=m.to_torch("down_w", l).view(d, s.d_ff).float(),
                ln1=m.to_torch("ln1", l).float(), ln2=m.to_torch("ln2", l).float()))
        self.feat_layers = (min(1, s.n_layers - 1), s.n_layers // 2, s.n_layers - 1)

    def mm(self, a, w):
        if self.bf16_mm:
            return (a.to(torch.bfloat16) @ w.to(torch.bfloat16).t()).float()
        return a @ w.t()

    def rms(self, x, w):
        return bf(x * torch.rsqrt((x * x).mean(-1, keepdim=True) + self.s.rms_eps) * w)

    def rope(self, x, pos):
        hd = self.s.head_dim
        half = hd // 2
        inv = torch.tensor([self.s.rope_theta ** (-2.0 * i / hd) for i in range(half)], dtype=torch.float64,
                           device=x.device)
        ang = pos.double()[:, None] * inv[None]
        c, sn = torch.cos(ang).float()[:, None], torch.sin(ang).float()[:, None]
        x1, x2 = x[..., :half], x[..., half:]
        return bf(torch.cat([x1 * c - x2 * sn, x2 * c + x1 * sn], -1))

    def attend(self, q, k, v):
        # q [T, H, hd], k/v [T, KV, hd]; causal
        T, H, hd = q.shape
        G = H // k.shape[1]
        k = k.repeat_interleave(G, 1)
        v = v.repeat_interleave(G, 1)
        sc = torch.einsum("thd,shd->hts", q, k) / hd ** 0.5
        mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=q.device), 1)
        sc = sc.masked_fill(mask, float("-inf"))
        p = torch.softmax(sc, -1)
        return bf(torch.einsum("hts,shd->thd", p, v))

    def layer(self, x, L, pos):
        s = self.s
        T = x.shape[0]
        h = self.rms(x, L["ln1"])
        qkv = bf(self.mm(h, L["qkv_w"]) + L["qkv_b"])
        H, KV, hd = s.n_heads, s.n_kv_heads, s.head_dim
        q = self.rope(qkv[:, :H * hd].view(T, H, hd), pos)
        k = self.rope(qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd), pos)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        ao = self.attend(q, k, v).reshape(T, H * hd)
        x = x + self.mm(ao, L["o_w"])
        h2 = self.rms(x, L["ln2"])
        mlp = bf(torch.nn.functional.silu(self.mm(h2, L["g_w"])) * self.mm(h2, L["u_w"]))
        return x + self.mm(mlp, L["down_w"])

    def forward(self, tokens, last_only=False):
        """Logits [T, V] for every position (last_only: [1, V] for the last position; the
        full-vocabulary rows at V ~ 152K are large) and the EAGLE features [T, 3, d]."""
        dev = self.emb.device
        tok = torch.tensor(tokens, device=dev)
        pos = torch.arange(len(tokens), device=dev)
        x = self.emb[tok].clone()
        feats = []
        for l, L in enumerate(self.layers):
            x = self.layer(x, L, pos)
            for f in self.feat_layers:
                if f == l:
                    feats.append(bf(x))
        if last_only:
            x = x[-1:]
        logits = self.mm(self.rms(x, self.final), self.emb) * self.s.logit_scale
        return logits, torch.stack(feats, 1)


class DrafterRef:
    """EAGLE-3-style drafter: f = fc([g_low, g_mid, g_high] at p-1), one layer over
    [RMSNorm(emb(x_p)), RMSNorm(f)], own LM head. q(. | x_0..x_p) is the row at position p."""

    def __init__(self, dm, target_ref):
        s = dm.shape
        d, q = s.d_model, (s.n_heads + 2 * s.n_kv_heads) * s.head_dim
        self.t = target_ref
        self.s = s
        self.fc = dm.to_torch("fc_w").view(d, 3 * d).float()
        self.ne = dm.to_torch("norm_emb").float()
        self.nh = dm.to_torch("norm_hid").float()
        gu = dm.to_torch("gu_w").view(2 * s.d_ff, d).float()
        self.L = dict(qkv_w=dm.to_torch("qkv_w").view(q, 2 * d).float(), qkv_b=dm.to_torch("qkv_b").float(),
                      o_w=dm.to_torch("o_w").view(d, s.n_heads * s.head_dim).float(),
                      g_w=gu[0::2], u_w=gu[1::2],
                      down_w=dm.to_torch("down_w").view(d, s.d_ff).float(), ln2=dm.to_torch("ln2").float())
        self.final = dm.to_torch("final_norm").float()
        self.lm = dm.to_torch("lm_w").view(s.vocab, d).float()

    def context_logits(self, tokens, last_only=False):
        """q rows for every prefix of `tokens` with target features (the depth-0 / catch-up
        path). Returns [T, V] where row p is q(. | tokens[:p+1]) ([1, V] with last_only)."""
        t = self.t
        _, feats = t.forward(tokens, last_only=True)
        T, d = len(tokens), self.s.d_model
        prev = torch.zeros(T, 3 * d, device=feats.device)
        prev[1:] = feats[:-1].reshape(T - 1, 3 * d)
        f = t.mm(prev, self.fc)
        return self._layer_logits(tokens, f, last_only)[0]

    def _layer_logits(self, tokens, f, last_only=False):
        t, s = self.t, self.s
        dev = f.device
        tok = torch.tensor(tokens, device=dev)
        pos = torch.arange(len(tokens), device=dev)
        e = t.emb[tok]
        h = torch.cat([t.rms(e, self.ne), t.rms(f, self.nh)], -1)
        L = self.L
        T = len(tokens)
        H, KV, hd = s.n_heads, s.n_kv_heads, s.head_dim
        qkv = bf(t.mm(h, L["qkv_w"]) + L["qkv_b"])
        q = t.rope(qkv[:, :H * hd].view(T, H, hd), pos)
        k = t.rope(qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd), pos)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        x = f + t.mm(t.attend(q, k, v).reshape(T, H * hd), L["o_w"])
        h2 = t.rms(x, L["ln2"])
        x = x + t.mm(bf(torch.nn.functional.silu(t.mm(h2, L["g_w"])) * t.mm(h2, L["u_w"])), L["down_w"])
        y = x[-1:] if last_only else x
        return t.mm(t.rms(y, self.final), self.lm) * t.s.logit_scale, x
