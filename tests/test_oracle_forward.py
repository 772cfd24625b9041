"""Pins for oracle O1 (the numeric forward) against things other than itself.

* a library implementation: HF transformers LlamaForCausalLM (fp32, CPU) with
  the LoRA delta merged into W (W + s*B@A) — pins RoPE layout, eps placement,
  GQA grouping, SiLU, residual order (SURVEY.md §8(c) "What pins each part");
* brute force: a float64 scalar-loop forward on a micro model;
* closed forms: RoPE at position 0 is the identity and preserves pair norms;
  causal attention with S=1 returns V; RMSNorm of a constant vector; LoRA with
  B=0 is the base; L=0 reduces to W_head . RMSNorm(E[tok_last]);
* sensitivity: dropping the adapter moves the logits far beyond 2e-2.
"""
import math

import numpy as np
import pytest

import synth
from oracle import forward as F


def _hf_logits(cfg, w, tokens, adapter=None, mask=0, scale=1.0):
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    hc = tr.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model,
                        intermediate_size=cfg.d_ff, num_hidden_layers=cfg.n_layers,
                        num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_kv_heads,
                        rms_norm_eps=cfg.rms_eps, tie_word_embeddings=cfg.tie_embeddings,
                        rope_parameters={"rope_type": "default", "rope_theta": cfg.rope_theta},
                        max_position_embeddings=8192, attention_bias=False, mlp_bias=False)
    model = tr.LlamaForCausalLM(hc).float().eval()
    sd = {}
    for k in model.state_dict():
        name = k
        if cfg.tie_embeddings and k == "lm_head.weight":
            name = "model.embed_tokens.weight"
        W = np.asarray(w(name), dtype=np.float64)
        if adapter is not None and k.endswith("_proj.weight"):
            t = k.split(".")[-2][:-5]
            if (mask >> synth.TARGETS.index(t)) & 1:
                m = k[: -len(".weight")]
                W = W + scale * (np.asarray(adapter(m + ".lora_B"), np.float64)
                                 @ np.asarray(adapter(m + ".lora_A"), np.float64))
        sd[k] = torch.tensor(W, dtype=torch.float32)
    model.load_state_dict(sd, strict=False)
    with torch.no_grad():
        out = model(torch.tensor(tokens[None, :].astype(np.int64))).logits[0]
    return out.numpy().astype(np.float64)


@pytest.mark.parametrize("cfg,S,lora", [
    (synth.config("tiny"), 16, True),
    (synth.config("tiny"), 16, False),
    (synth.ModelConfig("gqa", 3, 256, 8, 2, 512, 512, rope_theta=500000.0), 33, True),
    (synth.ModelConfig("tied", 2, 128, 2, 1, 256, 300, tie_embeddings=True), 9, True),
])
def test_forward_matches_hf_llama(cfg, S, lora):
    w = F.synth_weights(cfg, 7)
    a = F.synth_adapter(cfg, 8, 11) if lora else None
    mask = 0x7F if lora else 0
    tok = synth.prompt(cfg, S, 3)
    ours = F.forward(cfg, w, tok, a, mask, 1.0, dtype=np.float64, all_logits=True)
    ref = _hf_logits(cfg, w, tok, a, mask, 1.0)
    assert np.abs(ours["logits_all"] - ref).max() < 1e-4
    assert ours["token"] == int(np.argmax(ref[-1]))


# ----------------------------------------------------------------------------
# brute force: scalar loops, float64, micro model
# ----------------------------------------------------------------------------
def _brute(cfg, w, a, mask, s, tok):
    d, H, KV, hd, F_ = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff
    S = len(tok)
    g = lambda n: np.asarray(w(n), np.float64)

    def lin(x, name, layer, t):
        W = g(name)
        out_dim, in_dim = W.shape
        y = [sum(x[c] * W[o, c] for c in range(in_dim)) for o in range(out_dim)]
        if a is not None and (mask >> synth.TARGETS.index(t)) & 1:
            m = synth.module_name(layer, t)
            A, B = np.asarray(a(m + ".lora_A"), np.float64), np.asarray(a(m + ".lora_B"), np.float64)
            tt = [sum(x[c] * A[j, c] for c in range(in_dim)) for j in range(A.shape[0])]
            for o in range(out_dim):
                y[o] += s * sum(tt[j] * B[o, j] for j in range(A.shape[0]))
        return y

    def norm(x, gn):
        ms = sum(v * v for v in x) / len(x)
        r = 1.0 / math.sqrt(ms + cfg.rms_eps)
        return [gn[i] * x[i] * r for i in range(len(x))]

    X = [list(g("model.embed_tokens.weight")[t]) for t in tok]
    for i in range(cfg.n_layers):
        p = f"model.layers.{i}."
        q, k, v = [], [], []
        for pos in range(S):
            xn = norm(X[pos], g(p + "input_layernorm.weight"))
            qq = lin(xn, p + "self_attn.q_proj.weight", i, "q")
            kk = lin(xn, p + "self_attn.k_proj.weight", i, "k")
            vv = lin(xn, p + "self_attn.v_proj.weight", i, "v")
            for vec, nh in ((qq, H), (kk, KV)):
                for h in range(nh):
                    for j in range(hd // 2):
                        ang = pos * cfg.rope_theta ** (-2.0 * j / hd)
                        x1, x2 = vec[h * hd + j], vec[h * hd + j + hd // 2]
                        vec[h * hd + j] = x1 * math.cos(ang) - x2 * math.sin(ang)
                        vec[h * hd + j + hd // 2] = x2 * math.cos(ang) + x1 * math.sin(ang)
            q.append(qq); k.append(kk); v.append(vv)
        for pos in range(S):
            o = [0.0] * (H * hd)
            for h in range(H):
                gk = h // (H // KV)
                sc = [sum(q[pos][h * hd + c] * k[j][gk * hd + c] for c in range(hd)) / math.sqrt(hd)
                      for j in range(pos + 1)]
                mx = max(sc)
                e = [math.exp(z - mx) for z in sc]
                den = sum(e)
                for c in range(hd):
                    o[h * hd + c] = sum(e[j] * v[j][gk * hd + c] for j in range(pos + 1)) / den
            oo = lin(o, p + "self_attn.o_proj.weight", i, "o")
            X[pos] = [X[pos][c] + oo[c] for c in range(d)]
        for pos in range(S):
            hn = norm(X[pos], g(p + "post_attention_layernorm.weight"))
            gg = lin(hn, p + "mlp.gate_proj.weight", i, "gate")
            uu = lin(hn, p + "mlp.up_proj.weight", i, "up")
            hh = [gg[j] / (1.0 + math.exp(-gg[j])) * uu[j] for j in range(F_)]
            dd = lin(hh, p + "mlp.down_proj.weight", i, "down")
            X[pos] = [X[pos][c] + dd[c] for c in range(d)]
    h = norm(X[-1], g("model.norm.weight"))
    Wh = g("model.embed_tokens.weight" if cfg.tie_embeddings else "lm_head.weight")
    return np.array([sum(Wh[r, c] * h[c] for c in range(d)) for r in range(Wh.shape[0])])


def test_forward_matches_scalar_brute_force():
    cfg = synth.ModelConfig("micro", 2, 16, 2, 1, 24, 40)
    w, a = F.synth_weights(cfg, 1), F.synth_adapter(cfg, 4, 2)
    tok = synth.prompt(cfg, 5, 9)
    ours = F.forward(cfg, w, tok, a, 0x7F, 0.5, dtype=np.float64)["logits"]
    ref = _brute(cfg, w, a, 0x7F, 0.5, tok)
    assert np.abs(ours - ref).max() < 1e-10


# ----------------------------------------------------------------------------
# closed forms
# ----------------------------------------------------------------------------
def test_rope_position_zero_identity_and_norm_preserving():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((6, 3, 64))
    cos, sin = F.rope_cos_sin(6, 64, 1e4, np.float64)
    y = F.rope(x, cos, sin)
    assert np.array_equal(y[0], x[0])
    pair = lambda z: z[..., :32] ** 2 + z[..., 32:] ** 2
    assert np.allclose(pair(y), pair(x), rtol=1e-12)


def test_attention_single_token_returns_v():
    rng = np.random.default_rng(1)
    q, k, v = rng.standard_normal((1, 4, 8)), rng.standard_normal((1, 2, 8)), rng.standard_normal((1, 2, 8))
    o = F.causal_attention(q, k, v).reshape(1, 4, 8)
    for h in range(4):
        assert np.allclose(o[0, h], v[0, h // 2])


def test_attention_first_row_is_causal():
    rng = np.random.default_rng(2)
    q, k, v = (rng.standard_normal((5, 2, 8)) for _ in range(3))
    o = F.causal_attention(q, k, v).reshape(5, 2, 8)
    assert np.allclose(o[0], v[0])          # position 0 sees only itself


def test_rmsnorm_constant_vector():
    x = np.full((1, 64), -3.0)
    g = np.linspace(0.5, 1.5, 64)
    y = F.rmsnorm(x, g, 0.0)
    assert np.allclose(y, -g)


def test_lora_zero_b_is_base_and_merged_identity():
    cfg = synth.config("tiny")
    w, a = F.synth_weights(cfg, 0), F.synth_adapter(cfg, 8, 0)
    tok = synth.prompt(cfg, 8, 0)
    zero_b = lambda n: np.zeros_like(a(n)) if n.endswith("lora_B") else a(n)
    r0 = F.forward(cfg, w, tok, dtype=np.float64)["logits"]
    rz = F.forward(cfg, w, tok, zero_b, 0x7F, 1.0, dtype=np.float64)["logits"]
    assert np.abs(r0 - rz).max() < 1e-12

    def merged(n):
        W = np.asarray(w(n), np.float64)
        if n.endswith("_proj.weight"):
            m = n[: -len(".weight")]
            W = W + np.asarray(a(m + ".lora_B"), np.float64) @ np.asarray(a(m + ".lora_A"), np.float64)
        return W
    rs = F.forward(cfg, w, tok, a, 0x7F, 1.0, dtype=np.float64)["logits"]
    rm = F.forward(cfg, merged, tok, dtype=np.float64)["logits"]
    assert np.abs(rs - rm).max() < 1e-10


def test_zero_layers_is_head_of_embedding():
    cfg = synth.config("tiny")
    w = F.synth_weights(cfg, 5)
    tok = synth.prompt(cfg, 4, 5)
    r = F.forward(cfg, w, tok, dtype=np.float64, n_layers=0)["logits"]
    e = np.asarray(w("model.embed_tokens.weight"), np.float64)[tok[-1]]
    g = np.asarray(w("model.norm.weight"), np.float64)
    h = g * e / math.sqrt(float(np.mean(e * e)) + 1e-5)
    assert np.allclose(r, np.asarray(w("lm_head.weight"), np.float64) @ h, atol=1e-12)


def test_adapter_is_detectable():
    cfg = synth.config("tiny")
    w, a = F.synth_weights(cfg, 0), F.synth_adapter(cfg, 8, 0)
    tok = synth.prompt(cfg, 16, 0)
    r0 = F.forward(cfg, w, tok)["logits"]
    r1 = F.forward(cfg, w, tok, a, 0x7F, 1.0)["logits"]
    assert np.abs(r0 - r1).max() > 0.2       # >> the 2e-2 parity tolerance


def test_fp32_close_to_fp64():
    cfg = synth.config("tiny")
    w, a = F.synth_weights(cfg, 4), F.synth_adapter(cfg, 8, 4)
    tok = synth.prompt(cfg, 16, 4)
    r32 = F.forward(cfg, w, tok, a, 0x7F, 1.0, dtype=np.float32)["logits"]
    r64 = F.forward(cfg, w, tok, a, 0x7F, 1.0, dtype=np.float64)["logits"]
    assert np.abs(r32 - r64).max() < 1e-4


# ----------------------------------------------------------------------------
# decode: the reference the GPU decode is checked against is
# the oracle's causal forward over prompt ++ generated tokens; pin it to an
# independent incremental (KV-cached) decoder: HF transformers' greedy generate
# ----------------------------------------------------------------------------
def test_greedy_decode_matches_hf_generate():
    torch = pytest.importorskip("torch")
    tr = pytest.importorskip("transformers")
    cfg = synth.ModelConfig("gqa", 2, 256, 8, 2, 512, 512, rope_theta=500000.0)
    w = F.synth_weights(cfg, 5)
    a = F.synth_adapter(cfg, 8, 6)
    mask, scale, n_new = 0x7F, 0.5, 6
    prompt = synth.prompt(cfg, 11, 2)
    # oracle: greedy loop over the full causal forward
    seq = list(prompt)
    ours = []
    for _ in range(n_new):
        out = F.forward(cfg, w, np.array(seq), a, mask, scale, dtype=np.float64)
        ours.append(out["logits"])
        seq.append(out["token"])
    # HF: LoRA merged into the weights, greedy generate with the KV cache
    hc = tr.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model,
                        intermediate_size=cfg.d_ff, num_hidden_layers=cfg.n_layers,
                        num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_kv_heads,
                        rms_norm_eps=cfg.rms_eps, tie_word_embeddings=False,
                        rope_parameters={"rope_type": "default", "rope_theta": cfg.rope_theta},
                        max_position_embeddings=8192, attention_bias=False, mlp_bias=False)
    model = tr.LlamaForCausalLM(hc).float().eval()
    sd = {}
    for k in model.state_dict():
        W = np.asarray(w(k), dtype=np.float64)
        if k.endswith("_proj.weight"):
            m = k[: -len(".weight")]
            W = W + scale * (np.asarray(a(m + ".lora_B"), np.float64)
                             @ np.asarray(a(m + ".lora_A"), np.float64))
        sd[k] = torch.tensor(W, dtype=torch.float32)
    model.load_state_dict(sd, strict=False)
    with torch.no_grad():
        g = model.generate(torch.tensor(prompt[None, :].astype(np.int64)), max_new_tokens=n_new,
                           min_new_tokens=n_new, do_sample=False, use_cache=True,
                           output_scores=True, return_dict_in_generate=True,
                           pad_token_id=0, eos_token_id=None)
    hf_tokens = g.sequences[0, len(prompt):].numpy()
    assert list(hf_tokens) == seq[len(prompt):]
    for t in range(n_new):
        assert np.abs(g.scores[t][0].numpy().astype(np.float64) - ours[t]).max() < 1e-4



# ---- bf16-emulation mode (SURVEY.md §8(c) O1 debug aid) ----
def test_round_bf16_matches_torch_and_ties_to_even():
    """round_bf16 against torch's own float32 -> bfloat16 conversion (RNE), and
    the tie cases by hand: 1 + 2^-8 -> 1 (even), 1 + 3 * 2^-8 -> 1 + 2^-6."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-6, 6, 20000),
                        np.float32([0.0, -0.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 65504.0])])
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(F.round_bf16(x), ref)
    assert F.round_bf16(np.float32([1 + 2 ** -8]))[0] == 1.0
    assert F.round_bf16(np.float32([1 + 3 * 2 ** -8]))[0] == 1 + 2 ** -6
    y = F.round_bf16(x)
    assert np.array_equal(F.round_bf16(y), y)                   # idempotent


def test_bf16_emulated_attention_closed_forms():
    """S = 1: P = 1 exactly, O = v; a row attending to one key is that key's v
    (the rounding of P and the fp32 row sum cancel)."""
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((1, 2, 64)).astype(np.float32) for _ in range(3))
    assert np.array_equal(F.causal_attention(q, k[:, :1], v[:, :1], p_bf16=True),
                          np.repeat(v[:, :1], 2, axis=1).reshape(1, -1))


def test_bf16_emulated_forward_within_bf16_envelope():
    """The emulated forward differs from fp32 (rounding points active) but stays
    inside the bf16 error envelope the GPU is held to (2e-2, north_star)."""
    cfg = synth.config("tiny")
    w = F.synth_weights(cfg, 0)
    tok = synth.prompt(cfg, 24, 2)
    a = F.synth_adapter(cfg, 8, 3)
    r32 = F.forward(cfg, w, tok, a, 0x7F, 1.0)
    r16 = F.forward(cfg, w, tok, a, 0x7F, 1.0, bf16_emulate=True)
    gap = float(np.abs(r32["logits"] - r16["logits"]).max())
    assert 1e-4 < gap < 2e-2, gap
