"""Decode profiling driver: 13B-shaped model, fully resident template, prompt
S, rank-16 LoRA; one prefill then N greedy decode steps (run under ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2503_06421_b200 import build  # noqa: E402

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="13b")
ap.add_argument("--S", type=int, default=2048)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--rank", type=int, default=16)
args = ap.parse_args()
cfg = synth.config(args.config)
tensors, fill = synth.model_inputs(cfg, 0)
cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
          n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
          rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps)
model = T.Model(cd, tensors, "base:0", fill=fill)
tpl = T.Template(model, T.Trace(model), T.template_opts(resident_bytes=T.U64_MAX,
                                                        max_tokens=args.S, device=0))
tpl.enable_decode(args.steps)
ad = None
if args.rank:
    slots, total = tpl.adapter_layout(args.rank, 0x7F)
    buf = T.PinnedBuffer(total)
    synth.adapter_fill(cfg, args.rank, 1, slots, buf.view(), 0x7F)
    ad = T.Adapter(tpl, args.rank, 1.0, 0x7F, buf, total, "adapter:1")
tokens = synth.prompt_fast(cfg, args.S, 0)
for _ in range(2):
    tpl.invoke(tokens, ad, want_logits=False)
    toks, _, st = tpl.decode(args.steps, ad, want_logits=False)
print("decode", st)
