"""Microbenchmark of the tcgen05 GEMM family at the 13B prefill shapes through
the per-op C-ABI entry (tidal_k_gemm), sweeping tile width / CTA group /
multicast clusters.  Each measurement launches the same GEMM REPS times back to
back (TIDAL_K_REPEAT) between two CUDA events; prints TF/s per variant.

    python tools/gemm_bench.py [--reps 20] [--S 2048]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_06421_b200 import build  # noqa: E402

build.build()
from paper_2503_06421_b200 import tidal as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--S", type=int, default=2048)
ap.add_argument("--lora", type=int, default=16)
ap.add_argument("--mc-sweep", action="store_true", help="residual GEMMs, mc 1 vs 2")
ap.add_argument("--small-sweep", action="store_true", help="all bn x cg x split-K variants")
ap.add_argument("--resid-sweep", action="store_true",
                help="O/down only: bn x split-K grid, 3 interleaved passes, median")
args = ap.parse_args()
M, r = args.S, args.lora
d, F = 5120, 13824


def rnd(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def bench(name, epi, bn, cg, mc, N_list, K, flops, ks=0, tail=0):
    code = epi | (bn << 8) | (cg << 20) | (mc << 22) | (ks << 24) | (tail << 28)
    A = rnd(M, K)
    srcs = N_list * 2 if epi == 2 else N_list  # EPI_SILU: gate and up
    Ws = [rnd(n, K, scale=1 / math.sqrt(K)) for n in srcs]
    Ts = [rnd(M, r) for _ in srcs] if r else None
    Bs = [rnd(n, r, scale=0.1) for n in srcs] if r else None
    if epi == 2:
        out = torch.zeros(M, N_list[0], dtype=torch.bfloat16, device="cuda")
        ldo, seg = N_list[0], [N_list[0]]
    elif epi == 3:
        out = torch.zeros(M, N_list[0], dtype=torch.float32, device="cuda")
        ldo, seg = N_list[0], N_list
    else:
        ldo = sum(N_list)
        out = torch.zeros(M, ldo, dtype=torch.bfloat16, device="cuda")
        seg = N_list
    rope = torch.zeros(M, 64, 2, dtype=torch.float32, device="cuda") if epi == 1 else None
    os.environ["TIDAL_K_REPEAT"] = "2"
    T.k_gemm(code, A, Ws, seg, out, ldo, M, K, Ts, Bs, r, rope, 128)  # warm
    os.environ["TIDAL_K_REPEAT"] = str(args.reps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        T.k_gemm(code, A, Ws, seg, out, ldo, M, K, Ts, Bs, r, rope, 128)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / args.reps)
    os.environ["TIDAL_K_REPEAT"] = "1"
    print(f"{name:8s} bn={bn:3d} cg={cg} mc={mc} ks={ks} tail={tail}  {best * 1e3:8.1f} us  "
          f"{flops / best / 1e9:7.0f} TF/s", flush=True)


if args.mc_sweep:  # CTA-pair clusters sharing the A tile (TMA multicast), residual GEMMs
    for name, N, K in (("o", d, d), ("down", d, F)):
        for bn in (192, 256):
            for mc in (1, 2):
                for ks in (1, 2, 3):
                    bench(name, 3, bn, 2, mc, [N], K, 2.0 * M * N * K, ks)
    sys.exit(0)

if args.small_sweep:  # every (bn, cg, ks) for the given S (short prompts)
    for name, epi, N, K, bns in (("qkv", 1, [d, d, d], d, (128, 256)), ("gate_up", 2, [F], d, (128,)),
                                 ("o", 3, [d], d, (128, 192, 256)), ("down", 3, [d], F, (128, 192, 256))):
        for bn in bns:
            for cg in (1, 2):
                for ks in ((0,) if epi != 3 else (1, 2, 3, 4)):
                    bench(name, epi, bn, cg, 1, N, K, 2.0 * M * sum(N) * K * (2 if epi == 2 else 1), ks)
    sys.exit(0)

if args.resid_sweep:
    import statistics
    res = {}
    for _ in range(3):
        for name, N, K in (("o", d, d), ("down", d, F)):
            for bn in (192, 256):
                for ks, tail in ((1, 0), (2, 0), (3, 0), (4, 0), (2, 1), (4, 1), (6, 1), (8, 1)):
                    import io, contextlib
                    buf = io.StringIO()
                    with contextlib.redirect_stdout(buf):
                        bench(name, 3, bn, 2, 1, [N], K, 2.0 * M * N * K, ks, tail)
                    us = float(buf.getvalue().split("us")[0].split()[-1])
                    res.setdefault((name, bn, ks, tail), []).append(us)
            import io, contextlib
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                bench(name, 3, 0, 0, 0, [N], K, 2.0 * M * N * K)   # the planner's choice
            us = float(buf.getvalue().split("us")[0].split()[-1])
            res.setdefault((name, "auto"), []).append(us)
    for k, v in sorted(res.items(), key=str):
        print(k, "median us", round(statistics.median(v), 1), [round(x, 1) for x in v])
    sys.exit(0)

shapes = [
    ("qkv", 1, [d, d, d], d, [256]),
    ("o", 3, [d], d, [192, 256]),
    ("gate_up", 2, [F], d, [128]),
    ("down", 3, [d], F, [192, 256]),
]
for name, epi, N_list, K, bns in shapes:
    Ntot = sum(N_list) * (2 if epi == 2 else 1)
    flops = 2.0 * M * Ntot * K
    for bn in bns:
        for ks in ((0, 1, 2, 3, 4, 5, 6) if epi == 3 else (0,)):
            bench(name, epi, bn, 2, 1, N_list, K, flops, ks)
