"""O1 — plain CPU forward of the Llama-style decoder (TEST INFRASTRUCTURE ONLY).

The paper runs stock PyTorch Llama functions (§7.1:
"Llama2-7B/13B, Llama3-8B ... with LoRA"); its method (§5.2)
only changes WHEN weights arrive, never WHAT is computed ("reducing TTFT ... to
the latency of either loading or inference").  So this oracle is the plain
definition of the first-token forward, written out step by step in the order
of SURVEY.md §8(c) O1, with the readings of DESIGN.md §Readings (A1 eps=1e-5,
HF rotate-half RoPE, GQA h -> h // (H/KV); A3 LoRA on all 7 projections with
scale s; A4 logits of the last position; A5 argmax lowest index on ties).

Arithmetic is numpy in ``dtype`` (float32 by default, as BASELINE.json
north_star fixes "a plain CPU fp32 forward pass"; float64 for the tight pins).
Weights arrive as bf16 and are upcast exactly.  No blocking, fusion or
reordering beyond the definition: every projection is one matmul, attention is
a per-head loop over the full causal score matrix.
"""
from __future__ import annotations

import math
from typing import Callable, Dict, Optional

import numpy as np

import synth

WeightFn = Callable[[str], np.ndarray]


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round to the nearest bf16, ties to even (the storage format of the GPU's
    activations), returned in x's dtype.  Used only by the bf16-emulation mode
    (SURVEY.md §8(c) O1 "bf16-emulated ... rounds (RNE) exactly where the GPU
    stores bf16"); finite inputs only."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32).astype(np.asarray(x).dtype)


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    """RMSNorm(x; g) = g * x / sqrt(mean(x^2) + eps)."""
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return g * (x / np.sqrt(ms + x.dtype.type(eps)))


def rope_cos_sin(n_pos: int, head_dim: int, theta: float, dtype) -> tuple:
    """inv_freq_i = theta^(-2i/hd), angle = pos * inv_freq_i, computed in
    float64 then cast (reading A1)."""
    i = np.arange(head_dim // 2, dtype=np.float64)
    inv_freq = theta ** (-(2.0 * i) / head_dim)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv_freq[None, :]
    return np.cos(ang).astype(dtype), np.sin(ang).astype(dtype)


def rope(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """HF rotate-half on x [S, n_heads, hd]: pairs (i, i + hd/2)."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray,
                     p_bf16: bool = False) -> np.ndarray:
    """O_h = softmax(Q_h K_g^T / sqrt(hd) + causal) V_g, g = h // (H/KV).
    q [S,H,hd], k/v [S,KV,hd] -> [S, H*hd].  p_bf16 (bf16 emulation): the
    unnormalised P = exp(s - max) is rounded to bf16 before P V and the fp32
    row sum of the unrounded P divides afterwards (FA-style)."""
    S, H, hd = q.shape
    KV = k.shape[1]
    grp = H // KV
    scale = q.dtype.type(1.0 / math.sqrt(hd))
    mask = np.triu(np.ones((S, S), dtype=bool), k=1)          # j > i is masked
    out = np.empty((S, H, hd), dtype=q.dtype)
    for h in range(H):
        g = h // grp
        s = (q[:, h, :] @ k[:, g, :].T) * scale
        s[mask] = -np.inf
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        if p_bf16:
            out[:, h, :] = (round_bf16(p) @ v[:, g, :]) / p.sum(axis=1, keepdims=True)
            continue
        p = p / p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ v[:, g, :]
    return out.reshape(S, H * hd)


def linear(x: np.ndarray, W: np.ndarray, lora: Optional[tuple], scale: float,
           t_bf16: bool = False) -> np.ndarray:
    """y = x W^T + s (x A^T) B^T  — the LoRA branch kept separate (A3).
    t_bf16 (bf16 emulation): T = s x A^T is stored as bf16 before T B^T."""
    y = x @ W.T
    if lora is not None:
        A, B = lora
        if t_bf16:
            y = y + round_bf16(x.dtype.type(scale) * (x @ A.T)) @ B.T
        else:
            y = y + x.dtype.type(scale) * ((x @ A.T) @ B.T)
    return y


def silu(x: np.ndarray) -> np.ndarray:
    return x / (x.dtype.type(1.0) + np.exp(-x))


def forward(cfg: synth.ModelConfig, weight: WeightFn, tokens: np.ndarray,
            adapter: Optional[WeightFn] = None, target_mask: int = 0,
            scale: float = 1.0, dtype=np.float32, n_layers: Optional[int] = None,
            all_logits: bool = False, stats: Optional[dict] = None,
            bf16_emulate: bool = False) -> Dict[str, np.ndarray]:
    """First-token forward.

    weight(name)  -> weight in HF shape, any float dtype holding bf16 values.
    adapter(name) -> LoRA tensor ("<module>.lora_A"/"lora_B") or None.
    n_layers      -> run only the first n layers (bounded CPU samples).
    bf16_emulate  -> debug mode: round (RNE) to bf16 exactly where the GPU path
                     stores bf16 — Xn, Q/K/V after RoPE, P before P V, the
                     attention output, T = s x A^T, H = silu(G) * U; the residual
                     stream, G / U and the head stay fp32.
    Returns {"logits": [V] of the last position, "token": argmax (lowest index
    on ties, A5), "hidden": final residual [S, d]}.
    """
    L = cfg.n_layers if n_layers is None else n_layers
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    S = int(tokens.shape[0])
    W = lambda n: np.asarray(weight(n), dtype=dtype)
    eps = cfg.rms_eps

    def lora_of(layer: int, t: str):
        ti = synth.TARGETS.index(t)
        if adapter is None or not (target_mask >> ti) & 1:
            return None
        m = synth.module_name(layer, t)
        return (np.asarray(adapter(m + ".lora_A"), dtype=dtype),
                np.asarray(adapter(m + ".lora_B"), dtype=dtype))

    cos, sin = rope_cos_sin(S, hd, cfg.rope_theta, dtype)
    rb = round_bf16 if bf16_emulate else (lambda t: t)
    tb = bf16_emulate
    # X = E[tok]   (fp32 residual stream)
    X = W("model.embed_tokens.weight")[tokens]
    for i in range(L):
        p = f"model.layers.{i}."
        # attention block
        Xn = rb(rmsnorm(X, W(p + "input_layernorm.weight"), eps))
        Q = linear(Xn, W(p + "self_attn.q_proj.weight"), lora_of(i, "q"), scale, tb)
        K = linear(Xn, W(p + "self_attn.k_proj.weight"), lora_of(i, "k"), scale, tb)
        V = rb(linear(Xn, W(p + "self_attn.v_proj.weight"), lora_of(i, "v"), scale, tb))
        Q = rb(rope(Q.reshape(S, H, hd), cos, sin))
        K = rb(rope(K.reshape(S, KV, hd), cos, sin))
        O = rb(causal_attention(Q, K, V.reshape(S, KV, hd), p_bf16=bf16_emulate))
        X = X + linear(O, W(p + "self_attn.o_proj.weight"), lora_of(i, "o"), scale, tb)
        # MLP block
        Hn = rb(rmsnorm(X, W(p + "post_attention_layernorm.weight"), eps))
        G = linear(Hn, W(p + "mlp.gate_proj.weight"), lora_of(i, "gate"), scale, tb)
        U = linear(Hn, W(p + "mlp.up_proj.weight"), lora_of(i, "up"), scale, tb)
        X = X + linear(rb(silu(G) * U), W(p + "mlp.down_proj.weight"), lora_of(i, "down"), scale, tb)
        if stats is not None:
            stats.setdefault("residual_rms", []).append(float(np.sqrt(np.mean(X * X))))
    head_name = "model.embed_tokens.weight" if cfg.tie_embeddings else "lm_head.weight"
    Wh = W(head_name)
    g_f = W("model.norm.weight")
    if all_logits:
        logits_all = rmsnorm(X, g_f, eps) @ Wh.T
        logits = logits_all[-1]
    else:
        h = rmsnorm(X[-1:], g_f, eps)[0]
        logits = Wh @ h
        logits_all = None
    out = {"logits": logits, "token": int(np.argmax(logits)), "hidden": X}
    if logits_all is not None:
        out["logits_all"] = logits_all
    return out


# ----------------------------------------------------------------------------
# Input plumbing (not arithmetic): seeded synthetic weights from ``synth``.
# ----------------------------------------------------------------------------
def synth_weights(cfg: synth.ModelConfig, seed: int, fast: bool = False,
                  keep: bool = True) -> WeightFn:
    """name -> float32 array of the seeded bf16 weight (lazy; cached if keep)."""
    specs = {s.name: s for s in synth.base_tensors(cfg)}
    cache: Dict[str, np.ndarray] = {}

    def get(name: str) -> np.ndarray:
        if name in cache:
            return cache[name]
        s = specs[name]
        bits = synth.tensor_bits_fast(s, synth.NS_BASE, seed) if fast else \
            synth.tensor_bits(s, synth.NS_BASE, seed)
        w = synth.bf16_bits_to_f32(bits)
        if keep:
            cache[name] = w
        return w
    return get


def synth_adapter(cfg: synth.ModelConfig, rank: int, seed: int, target_mask: int = 0x7F,
                  fast: bool = False) -> WeightFn:
    specs = {s.name: s for s in synth.adapter_tensors(cfg, rank, target_mask)}
    cache: Dict[str, np.ndarray] = {}

    def get(name: str) -> np.ndarray:
        if name not in cache:
            s = specs[name]
            bits = synth.tensor_bits_fast(s, synth.NS_ADAPTER, seed) if fast else \
                synth.tensor_bits(s, synth.NS_ADAPTER, seed)
            cache[name] = synth.bf16_bits_to_f32(bits)
        return cache[name]
    return get
