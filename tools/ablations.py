"""f2 ablations on one B200 (§7.3 fig:ttft-bs
lines 721-732, §7.4 tab:memory-merge lines 853-872), 13B shape, r16 LoRA:

  batch   TTFT of n prompts of 2048 tokens (weights streamed once) for
          n = 1, 2, 4, 8 at rho = 0 and at the Eq. 1 residency of n = 1:
          the turning point where compute overtakes the copy stream.
  merge   per_layer vs max_transfers=300 vs per_tensor ("No Merge") groups at
          rho = 0 for S = 512, 2048, 8192.

One JSON line per point to --out; L2 flushed before every invocation, median
of --reps device TTFTs.

    python tools/ablations.py [--only batch|merge] [--out gpurun_out/ablations.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2503_06421_b200 import build  # noqa: E402

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--only", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ablations.jsonl"))
args = ap.parse_args()

cfg = synth.config("13b")
r = 16
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(bench.cfg_dict(cfg), tensors, "base:0", fill=fill)
trace = T.Trace(model)
M = sum(s.nbytes for s in synth.base_tensors(cfg))
os.makedirs(os.path.dirname(args.out), exist_ok=True)
out = open(args.out, "a")


def emit(d):
    print(json.dumps(d), flush=True)
    out.write(json.dumps(d) + "\n")


def setup(policy, max_tokens):
    tpl = T.Template(model, trace, T.template_opts(resident_bytes=0, group_policy=policy,
                                                   max_tokens=max_tokens, device=0))
    slots, nb = tpl.adapter_layout(r, 0x7F)
    buf = T.PinnedBuffer(nb)
    synth.adapter_fill(cfg, r, 1, slots, buf.view(), 0x7F)
    return tpl, buf, nb


def timed(tpl, buf, nb, toks, debug=T.DEBUG_SCRUB_L2):
    ms, st = [], None
    for i in range(args.reps + 1):
        tpl.set_debug(debug)
        ad = T.Adapter(tpl, r, 1.0, 0x7F, buf, nb, "adapter:1")
        if toks.ndim == 2:
            _, _, st = tpl.invoke_batch(toks, ad, want_logits=False)
        else:
            _, _, st = tpl.invoke(toks, ad, want_logits=False)
        if i:
            ms.append(st["device_ms"])
    return statistics.median(ms), st


if args.only in (None, "batch"):
    S = 2048
    tpl, buf, nb = setup(0, 8 * S)
    one = synth.prompt_fast(cfg, S, 0)
    _, st = timed(tpl, buf, nb, one, T.DEBUG_SERIAL | T.DEBUG_SCRUB_L2)
    b_h2d = (st["bytes_streamed"] + st["bytes_adapter"]) / ((st["h2d_last_ms"] - st["h2d_first_ms"]) / 1e3)
    tpl.resize(T.template_opts(resident_bytes=T.U64_MAX))
    warm, _ = timed(tpl, buf, nb, one)
    for label, opts in (("rho0", T.template_opts(resident_bytes=0)),
                        ("eq1", T.template_opts(eq1=True, t_ttft_s=warm / 1e3, b_pcie_Bps=b_h2d))):
        tpl.resize(opts)
        for n in (1, 2, 4, 8):
            toks = synth.prompt_fast(cfg, n * S, 0).reshape(n, S)
            ms, st = timed(tpl, buf, nb, toks if n > 1 else toks[0])
            streamed = st["bytes_streamed"] + st["bytes_adapter"]
            t_pcie = streamed / b_h2d * 1e3
            t_tc = n * bench.prefill_flops(cfg, S, r, 1) / (bench.peaks()[0]["bf16_tflops"] * 1e12) * 1e3
            emit({"ablation": "batch", "residency": label, "rho": st["bytes_resident"] / M,
                  "n_prompts": n, "seq_len": S, "ttft_ms": ms, "ms_per_prompt": ms / n,
                  "t_pcie_ms": t_pcie, "t_tensor_ms": t_tc, "bound": "pcie" if t_pcie >= t_tc else "tensor",
                  "warm_rho1_ms_n1": warm, "b_h2d_GBps": b_h2d / 1e9})
    del tpl

if args.only in (None, "merge"):
    for policy, name in ((0, "per_layer"), (1, "max_transfers_300"), (2, "per_tensor")):
        tpl, buf, nb = setup(policy, 8192)
        for S in (512, 2048, 8192):
            toks = synth.prompt_fast(cfg, S, 0)
            ms, st = timed(tpl, buf, nb, toks)
            emit({"ablation": "merge", "policy": name, "seq_len": S, "rho": 0.0, "ttft_ms": ms,
                  "n_copies": st["n_copies"],
                  "h2d_span_ms": st["h2d_last_ms"] - st["h2d_first_ms"],
                  "copy_rate_GBps": (st["bytes_streamed"] + st["bytes_adapter"]) /
                  ((st["h2d_last_ms"] - st["h2d_first_ms"]) / 1e3) / 1e9})
        del tpl
