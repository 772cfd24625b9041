"""Warm (fully template-resident, rho = 1) prefill timing for quick A/B runs of
kernel variants selected by environment variables (one process per variant):

    TIDAL_FUSED_SHRINK=0 python tools/warm.py --seq 2048 --steps 10
    python tools/warm.py --profile        # + per-kernel-class event table

Prints one JSON line: mean / median device ms over the timed steps (L2 flushed
before each), and, with --profile, the per-class table of a separate pass.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2503_06421_b200 import build  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="13b")
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--rank", type=int, default=16)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--rho", type=float, default=1.0)
ap.add_argument("--profile", action="store_true")
ap.add_argument("--tag", default="")
args = ap.parse_args()

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

cfg = synth.config(args.config)
cd = dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
          n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab, rope_theta=cfg.rope_theta,
          rms_eps=cfg.rms_eps)
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(cd, tensors, "base:0", fill=fill)
trace = T.Trace(model)
M = sum(s.nbytes for s in synth.base_tensors(cfg))
tpl = T.Template(model, trace, T.template_opts(resident_bytes=int(args.rho * M) if args.rho < 1
                                               else T.U64_MAX, max_tokens=args.seq, device=0))
ad = None
if args.rank:
    slots, nb = tpl.adapter_layout(args.rank, 0x7F)
    buf = T.PinnedBuffer(nb)
    synth.adapter_fill(cfg, args.rank, 1, slots, buf.view(), 0x7F)
tok = synth.prompt_fast(cfg, args.seq, 0)


def step(dbg):
    tpl.set_debug(dbg)
    a = T.Adapter(tpl, args.rank, 1.0, 0x7F, buf, nb, "adapter:1") if args.rank else None
    t, _, st = tpl.invoke(tok, a, want_logits=False)
    return st["device_ms"], t


for _ in range(args.warmup):
    step(T.DEBUG_SCRUB_L2)
ms = [step(T.DEBUG_SCRUB_L2)[0] for _ in range(args.steps)]
out = {"tag": args.tag, "seq": args.seq, "rho": args.rho, "rank": args.rank,
       "mean_ms": statistics.mean(ms), "median_ms": statistics.median(ms), "min_ms": min(ms),
       "token": step(T.DEBUG_SCRUB_L2)[1],
       "env": {k: v for k, v in os.environ.items() if k.startswith("TIDAL_")}}
if args.profile:
    tpl.profile(reset=True)
    for _ in range(3):
        step(T.DEBUG_SCRUB_L2 | T.DEBUG_PROFILE)
    out["kernels_ms_per_step"] = {k: round(v["ms"] / 3, 3) for k, v in tpl.profile(reset=True).items()
                                  if v["launches"]}
    tpl.profile(reset=True)
    for _ in range(args.steps):
        step(T.DEBUG_SCRUB_L2 | T.DEBUG_PROFILE_GEMM)
    out["gemm_us_per_launch"] = {k: round(1e3 * v["ms"] / v["launches"], 1)
                                 for k, v in tpl.profile(reset=True).items() if v["launches"]}
print(json.dumps(out))
