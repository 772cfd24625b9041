"""Decode continuation against the oracle (GPU).

After a template-start prefill of S tokens, greedy decoding of n tokens: step
t feeds token x_t at position S + t and its logits must equal the oracle's
logits at position S + t of the full sequence prompt ++ [x_0 .. x_{n-1}]
(one causal oracle forward with all_logits gives every step's reference: the
definition of a KV-cached decode is exactly the causal forward over the
longer sequence).  Same tolerances as the prefill (max-abs 2e-2, token by the
margin rule, A6).  Covers: tiny (hd = 64) with LoRA and a partly
streamed template, the 13B width (hd = 128, reduced depth) with rank-16 LoRA,
GQA / theta = 5e5 (70B-like head layout, reduced width), repeated decodes
(graph replay from a fresh prefill), and the error paths.
"""
import numpy as np
import pytest

import synth
from oracle import forward as F

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL, MARGIN = 2e-2, 4e-2


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_06421_b200 import build
    build.build()
    from paper_2503_06421_b200 import tidal
    tidal.lib()
    return tidal


def _setup(T, cfg, S, rank, rho, max_new, seed=0):
    tensors, fill = synth.model_inputs(cfg, seed)
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    model = T.Model(cd, tensors, f"base:{seed}", fill=fill)
    trace = T.Trace(model)
    M = sum(s.nbytes for s in synth.base_tensors(cfg))
    tpl = T.Template(model, trace, T.template_opts(resident_bytes=int(rho * M), max_tokens=S,
                                                   device=0))
    tpl.enable_decode(max_new)
    ad = None
    if rank:
        slots, total = tpl.adapter_layout(rank, 0x7F)
        buf = T.PinnedBuffer(total)
        synth.adapter_fill(cfg, rank, seed + 1, slots, buf.view(), 0x7F)
        ad = T.Adapter(tpl, rank, 0.5, 0x7F, buf, total, f"adapter:{seed + 1}")
        ad._buf = buf
    return model, tpl, ad


def _check_steps(cfg, prompt, first, toks, logits, rank, seed=0):
    seq = np.concatenate([prompt, [first], toks[:-1]]).astype(np.int64)
    ref = F.forward(cfg, F.synth_weights(cfg, seed, fast=True, keep=False), seq,
                    F.synth_adapter(cfg, rank, seed + 1, fast=True) if rank else None,
                    0x7F if rank else 0, 0.5, all_logits=True)["logits_all"]
    S = len(prompt)
    worst = 0.0
    for t in range(len(toks)):
        r = ref[S + t]
        err = float(np.abs(logits[t] - r).max())
        worst = max(worst, err)
        assert err <= TOL, (t, err)
        top = np.sort(r)[-2:]
        if top[1] - top[0] > MARGIN:
            assert toks[t] == int(np.argmax(r)), t
        assert r[toks[t]] >= r.max() - MARGIN, t
    return worst


@pytest.mark.parametrize("cfg_name,over,S,rank,rho,n", [
    ("tiny", {}, 16, 8, 0.5, 12),
    ("tiny", {}, 37, 0, 0.0, 30),
    ("13b", {"n_layers": 2}, 130, 16, 0.5, 6),
    ("70b", {"n_layers": 2, "d_model": 2048, "n_heads": 16, "n_kv_heads": 2, "d_ff": 5632,
             "vocab": 4096}, 67, 16, 1.0, 5),
])
def test_decode_matches_oracle(T, cfg_name, over, S, rank, rho, n):
    cfg = synth.config(cfg_name, **over)
    model, tpl, ad = _setup(T, cfg, S, rank, rho, max_new=n + 3)
    prompt = synth.prompt_fast(cfg, S, 0)
    first, _, _ = tpl.invoke(prompt, ad)
    toks, logits, st = tpl.decode(n, ad)
    assert st["n_kernels"] > 0 and st["per_token_ms"] > 0
    _check_steps(cfg, prompt, first, toks, logits, rank)
    # a second prefill + decode replays the captured step graph: identical results
    first2, _, _ = tpl.invoke(prompt, ad)
    toks2, logits2, _ = tpl.decode(n, ad)
    assert first2 == first and np.array_equal(toks2, toks)
    assert np.array_equal(logits2, logits)
    del tpl, model


def test_decode_error_paths(T):
    cfg = synth.config("tiny")
    tensors, fill = synth.model_inputs(cfg, 0)
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    model = T.Model(cd, tensors, "base:0", fill=fill)
    tpl = T.Template(model, T.Trace(model), T.template_opts(max_tokens=32, device=0))
    prompt = synth.prompt(cfg, 8, 0)
    with pytest.raises(T.TidalError):  # not enabled
        tpl.decode(2)
    tpl.enable_decode(4)
    with pytest.raises(T.TidalError):  # no prefill since enabling
        tpl.decode(2)
    tpl.invoke(prompt)
    with pytest.raises(T.TidalError):  # beyond max_new_tokens
        tpl.decode(5)
    tpl.invoke_batch(np.stack([prompt, prompt]))
    with pytest.raises(T.TidalError):  # the last prefill was batched
        tpl.decode(2)
    tpl.invoke(prompt)
    toks, _, _ = tpl.decode(4, want_logits=False)
    assert toks.shape == (4,)


def test_decode_refuses_another_adapter(T):
    """decode must continue with the adapter of the preceding prefill,
    even when another adapter has the same rank and targets (same arena layout)."""
    cfg = synth.config("tiny")
    model, tpl, ad = _setup(T, cfg, 16, 8, 1.0, 4)
    slots, total = tpl.adapter_layout(8, 0x7F)
    buf = T.PinnedBuffer(total)
    synth.adapter_fill(cfg, 8, 9, slots, buf.view(), 0x7F)
    other = T.Adapter(tpl, 8, 0.5, 0x7F, buf, total, "adapter:9")
    prompt = synth.prompt(cfg, 16, 3)
    tpl.invoke(prompt, ad)
    with pytest.raises(T.TidalError):
        tpl.decode(2, other)
    with pytest.raises(T.TidalError):
        tpl.decode(2)            # nor without the adapter
    toks, _, _ = tpl.decode(2, ad, want_logits=False)
    assert toks.shape == (2,)
