"""Shape-space sweep on one B200 (BASELINE.json configs[1] and configs[4]).

One model and pinned pool per (config), then for each point: resize the
template (rho), attach the adapter (rank), invoke S tokens — L2 scrubbed
before every timed invocation, median of 3 device TTFTs — and its roofline
max(streamed bytes / B_h2d, FLOPs / bf16 peak), B_h2d measured on the same
template (fully streamed, load-then-infer).  One JSON line per point.

    python tools/sweep.py [--config 13b] [--out gpurun_out/sweep.jsonl]
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
ap.add_argument("--config", default="13b")
ap.add_argument("--S", type=int, nargs="*", default=None, help="override prompt lengths")
ap.add_argument("--rho", type=float, nargs="*", default=None, help="override resident fractions")
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
ap.add_argument("--eq1", action="store_true",
                help="template sized by Eq. 1 per S (warm TTFT measured first, adapter counted)")
args = ap.parse_args()

cfg = synth.config(args.config)
P, _ = bench.peaks()
if args.eq1:  # rho < 0: Eq. 1 (bench.py's rule, reading A7b)
    pts = [(S, 0 if args.config == "7b" else 16, -1.0) for S in (args.S or (256, 867, 1154, 2048, 4096, 8192))]
elif args.config == "7b":
    pts = [(2048, 0, rho) for rho in (0.0, 1.0)]
else:
    pts = [(S, 16, rho) for S in (args.S or (256, 867, 2048, 6101, 8192))
           for rho in (args.rho or (0.0, 0.5, 1.0))]
    if not args.S:
        pts += [(2048, r, rho) for r in (8, 32, 64) for rho in (0.0, 1.0)]
maxS = max(p[0] for p in pts)
tensors, fill = synth.model_inputs(cfg, 0)
model = T.Model(bench.cfg_dict(cfg), tensors, "base:0", fill=fill)
tpl = T.Template(model, T.Trace(model), T.template_opts(resident_bytes=0, max_tokens=maxS, device=0))
M = sum(s.nbytes for s in synth.base_tensors(cfg))
adapters = {}


def adapter(r):
    if not r:
        return None
    if r not in adapters:
        slots, total = tpl.adapter_layout(r, 0x7F)
        buf = T.PinnedBuffer(total)
        synth.adapter_fill(cfg, r, 1, slots, buf.view(), 0x7F)
        adapters[r] = (buf, total)
    buf, total = adapters[r]
    return T.Adapter(tpl, r, 1.0, 0x7F, buf, total, f"adapter:{r}")


def run(S, r, debug, n=3):
    toks = synth.prompt_fast(cfg, S, 0)
    out = []
    for i in range(n + 1):
        tpl.set_debug(debug)
        ad = adapter(r)
        _, _, st = tpl.invoke(toks, ad, want_logits=False)
        if i:
            out.append(st)
    return out


# B_h2d of this path: fully streamed, serial (copies alone on the copy stream)
tpl.resize(T.template_opts(resident_bytes=0))
st = run(2048 if maxS >= 2048 else maxS, 16 if args.config != "7b" else 0,
         T.DEBUG_SERIAL | T.DEBUG_SCRUB_L2, n=1)[0]
b_h2d = (st["bytes_streamed"] + st["bytes_adapter"]) / ((st["h2d_last_ms"] - st["h2d_first_ms"]) / 1e3)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "a") as f:
    for S, r, rho in pts:
        t_warm = None
        if rho < 0:  # Eq. 1: warm TTFT at this S, then M_prefetch = M + M_adapter - T x B
            tpl.resize(T.template_opts(resident_bytes=T.U64_MAX))
            t_warm = statistics.median(s["device_ms"] for s in run(S, r, T.DEBUG_SCRUB_L2))
            anb = adapters[r][1] if r else 0
            t_eq1 = bench.eq1_t_ttft(t_warm / 1e3, anb, b_h2d)
            tpl.resize(T.template_opts(eq1=True, t_ttft_s=t_eq1, b_pcie_Bps=b_h2d))
        else:
            tpl.resize(T.template_opts(resident_bytes=T.U64_MAX if rho >= 1 else int(rho * M)))
        sts = run(S, r, T.DEBUG_SCRUB_L2)
        ms = statistics.median(s["device_ms"] for s in sts)
        streamed = sts[0]["bytes_streamed"] + sts[0]["bytes_adapter"]
        flops = bench.prefill_flops(cfg, S, r, 1)
        t_pcie = streamed / b_h2d * 1e3
        t_tc = flops / (P["bf16_tflops"] * 1e12) * 1e3
        t_tc_sus = flops / (P.get("bf16_tflops_sustained", P["bf16_tflops"]) * 1e12) * 1e3
        w_bytes = sts[0]["bytes_streamed"] + sts[0]["bytes_resident"] + sts[0]["bytes_adapter"]
        t_hbm = w_bytes / (P["hbm_gbs"] * 1e9) * 1e3   # every weight read once from HBM
        roof = max(t_pcie, t_tc, t_hbm)
        bound = max((("pcie", t_pcie), ("tensor", t_tc), ("hbm", t_hbm)), key=lambda kv: kv[1])[0]
        line = {"config": args.config, "S": S, "lora_rank": r,
                "rho_requested": "eq1" if rho < 0 else rho, "t_warm_ms": t_warm,
                "rho_realized": sts[0]["bytes_resident"] / M, "ttft_ms": ms,
                "tokens_per_s": S / (ms / 1e3), "t_pcie_ms": t_pcie, "t_tensor_ms": t_tc,
                "t_tensor_sustained_ms": t_tc_sus, "t_hbm_ms": t_hbm, "roof_ms": roof,
                "bound": bound, "frac": roof / ms,
                "frac_sustained": max(t_pcie, t_tc_sus, t_hbm) / ms, "b_h2d_GBps": b_h2d / 1e9,
                "h2d_span_ms": statistics.median(s["h2d_last_ms"] - s["h2d_first_ms"] for s in sts),
                "compute_start_ms": statistics.median(s["compute_first_ms"] for s in sts)}
        print(json.dumps(line), flush=True)
        f.write(json.dumps(line) + "\n")
