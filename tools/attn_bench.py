"""Microbenchmark of the tcgen05 causal attention (hd = 128) at the 13B prefill
shape through the per-op C-ABI entry (tidal_k_attention_tc): REPS launches
back to back between two CUDA events (TIDAL_K_REPEAT), best of 3.

    python tools/attn_bench.py [--S 2048] [--H 40] [--reps 20]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_06421_b200 import build  # noqa: E402

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--S", type=int, nargs="+", default=[2048])
ap.add_argument("--H", type=int, default=40)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
for S in args.S:
    H = KV = args.H
    hd = 128
    qkv = torch.randn(S, (H + 2 * KV) * hd, device="cuda").to(torch.bfloat16)
    vt_ld = (S + 63) // 64 * 64
    vt = torch.randn(KV * hd, vt_ld, device="cuda").to(torch.bfloat16)
    O = torch.empty(S, H * hd, dtype=torch.bfloat16, device="cuda")
    os.environ["TIDAL_K_REPEAT"] = "2"
    T.k_attention_tc(qkv, vt, vt_ld, O, S, H, KV)
    os.environ["TIDAL_K_REPEAT"] = str(args.reps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        T.k_attention_tc(qkv, vt, vt_ld, O, S, H, KV)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / args.reps)
    os.environ["TIDAL_K_REPEAT"] = "1"
    flops = 2.0 * hd * H * S * (S + 1)  # causal QK^T + PV
    print(f"attention S={S} H={H}: {best * 1e3:7.1f} us  {flops / best / 1e9:6.0f} TF/s", flush=True)
