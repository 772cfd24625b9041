"""Parity across BASELINE.json configs[3]/[4]'s shape space (GPU, slow).

Reduced-depth models at full width (the kernels' tiling depends on width, S
and rank, not on depth): 13B width over prompt lengths that hit GEMM M-tails
and attention tails (Table 2's mean lengths 867/1154), LoRA
ranks 8..64 and resident fractions 0..1; the 70B shape (d=8192, GQA 64/8,
theta=5e5, V=128256).  Against the fp32 oracle: logits max-abs 2e-2, first
token by the margin rule.
"""
import numpy as np
import pytest

import synth
from oracle import forward as F

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

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


def _run(T, cfg, S, rank, rho, seed=0):
    tensors, fill = synth.model_inputs(cfg, seed)
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    model = T.Model(cd, tensors, f"base:{seed}", fill=fill)
    trace = T.Trace(model)
    M = sum(s.nbytes for s in synth.base_tensors(cfg))
    tpl = T.Template(model, trace, T.template_opts(resident_bytes=int(rho * M), max_tokens=S,
                                                   device=0))
    tpl.set_debug(T.DEBUG_POISON)
    ad = None
    if rank:
        slots, total = tpl.adapter_layout(rank, 0x7F)
        buf = T.PinnedBuffer(total)
        synth.adapter_fill(cfg, rank, seed + 1, slots, buf.view(), 0x7F)
        ad = T.Adapter(tpl, rank, 1.0, 0x7F, buf, total, f"adapter:{seed + 1}")
    tokens = synth.prompt_fast(cfg, S, seed)
    tok, logits, _ = tpl.invoke(tokens, ad)
    del tpl, model
    ref = F.forward(cfg, F.synth_weights(cfg, seed, fast=True, keep=False), tokens,
                    F.synth_adapter(cfg, rank, seed + 1, fast=True) if rank else None,
                    0x7F if rank else 0, 1.0)
    err = float(np.abs(logits - ref["logits"]).max())
    assert err <= TOL, err
    top = np.sort(ref["logits"])[-2:]
    if top[1] - top[0] > MARGIN:
        assert tok == ref["token"]
    assert ref["logits"][tok] >= ref["logits"].max() - MARGIN


@pytest.mark.parametrize("S,rank,rho", [
    (256, 8, 0.0), (867, 16, 0.5), (1154, 32, 1.0), (4096, 64, 0.25), (2048, 16, 0.75),
])
def test_13b_width_sweep(T, S, rank, rho):
    _run(T, synth.config("13b", n_layers=2), S, rank, rho)


def test_70b_shape(T):
    _run(T, synth.config("70b", n_layers=1), 512, 16, 0.5)
