"""Workload for compute-sanitizer (racecheck / synccheck on tiny):
the tiny config (hd 64) and a small hd-128 GQA config (tcgen05 attention), a
rank-8 LoRA attached, half the template streamed, eager and graph-replayed
invocations, checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from oracle import forward as F  # noqa: E402
from paper_2503_06421_b200 import tidal as T  # noqa: E402

for cfg in (synth.config("tiny"),
            synth.ModelConfig("gqa128", 2, 512, 4, 2, 1376, 2048, rope_theta=500000.0)):
    cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
              n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
              rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
    tensors, fill = synth.model_inputs(cfg, 0)
    model = T.Model(cd, tensors, "base:0", fill=fill)
    tok = synth.prompt(cfg, 200, 0)
    trace = T.Trace(model)
    M = sum(s.nbytes for s in synth.base_tensors(cfg))
    tpl = T.Template(model, trace, T.template_opts(resident_bytes=M // 2, max_tokens=256, device=0))
    slots, total = tpl.adapter_layout(8, 0x7F)
    buf = T.PinnedBuffer(total)
    synth.adapter_fill(cfg, 8, 0, slots, buf.view())
    ad = T.Adapter(tpl, 8, 1.0, 0x7F, buf, total, "adapter:0")
    ref = F.forward(cfg, F.synth_weights(cfg, 0), tok, F.synth_adapter(cfg, 8, 0), 0x7F, 1.0)
    for dbg in (T.DEBUG_NO_GRAPH | T.DEBUG_POISON, T.DEBUG_POISON, 0):
        tpl.set_debug(dbg)
        token, logits, st = tpl.invoke(tok, ad)
        err = float(np.abs(logits - ref["logits"]).max())
        print(f"{cfg.name} debug={dbg}: token {token} (oracle {ref['token']}) err {err:.2e} "
              f"kernels {st['n_kernels']}", flush=True)
        assert err <= 2e-2
print("sanitize workload ok")
