"""13B-width, 2-layer prefill at S=2048 with a rank-16 LoRA (the stream-K QKV
tail is active at this shape) against the oracle; used under compute-sanitizer."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import forward as F  # noqa: E402
from paper_2503_06421_b200 import tidal as T  # noqa: E402

S = int(os.environ.get("SK_S", "2048"))
cfg = synth.config("13b", n_layers=2)
cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads,
          d_ff=cfg.d_ff, vocab=cfg.vocab, rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(cd, tensors, "base:0", fill=fill)
tpl = T.Template(model, T.Trace(model), T.template_opts(max_tokens=S, device=0))
slots, nb = tpl.adapter_layout(16, 0x7F)
buf = T.PinnedBuffer(nb)
synth.adapter_fill(cfg, 16, 1, slots, buf.view(), 0x7F)
ad = T.Adapter(tpl, 16, 0.5, 0x7F, buf, nb, "adapter:1")
tok = synth.prompt_fast(cfg, S, 3)
tpl.set_debug(T.DEBUG_NO_GRAPH)
t, lg, st = tpl.invoke(tok, ad)
ref = F.forward(cfg, F.synth_weights(cfg, 0, fast=True, keep=False), tok,
                F.synth_adapter(cfg, 16, 1, fast=True), 0x7F, 0.5)
err = float(np.abs(lg - ref["logits"]).max())
print("token", t, ref["token"], "err", err)
assert err < 2e-2
