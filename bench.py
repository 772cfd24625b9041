"""bench.py — template-start TTFT of a Llama2-13B-shaped prefill with a
dynamically attached rank-16 LoRA (BASELINE.json configs[2], the paper's
Fig. 1 workload: 2k-token prompt), on N B200s (N>1: tensor parallel, each
rank streams its own shard over its own PCIe link; NCCL allreduce over NVLink).

One timed step = attach the adapter (host) + one tidal_invoke_prefill: the
non-resident weights and the adapter stream from the pinned host pool in
traced order while the prefill runs, gated by per-group events; the step ends
with the first token and the last-position logits on the host.  The template
size is set by the paper's Eq. 1 from the warm TTFT and the H2D bandwidth
measured in this same run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tidal|reference]
                    [--config 13b] [--seq 2048] [--rank 16] [--rho eq1|<fraction>]

Prints ONE JSON line (rank 0).  value = mean device TTFT (ms, lower is better).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def cfg_dict(cfg):
    return dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
                n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
                rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps,
                tie_embeddings=cfg.tie_embeddings)


def prefill_flops(cfg, S, r, world):
    """Algorithmic prefill FLOPs per rank: 2*S per linear parameter, causal
    attention 2*hd*H*S*(S+1) per layer, LoRA 2*S*r*(in+out) per target, head
    2*d*V for the last position."""
    d, F, hd = cfg.d_model, cfg.d_ff, cfg.head_dim
    nq, nkv = cfg.n_heads * hd, cfg.n_kv_heads * hd
    lin = d * (nq + 2 * nkv) + nq * d + 3 * d * F
    lora = r * ((d + nq) + 2 * (d + nkv) + (nq + d) + 2 * (d + F) + (F + d)) if r else 0
    per_layer = 2 * S * lin + 2 * hd * cfg.n_heads * S * (S + 1) + 2 * S * lora
    return (cfg.n_layers * per_layer + 2 * d * cfg.vocab) / world


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.rows, self.p = dev, [], None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


ORACLE_LAYERS = 3   # decoder layers per bounded oracle sample (+ embed and head)


def oracle_sampler(cfg, S, r, seed=0, n_layers=ORACLE_LAYERS):
    """A bounded oracle sample: embed + the first n_layers decoder layers +
    head at full width and full S, LoRA on all 7 targets.  Inputs (weights,
    adapter, prompt) are generated once, outside any timing; the returned
    callable times one forward and returns seconds."""
    from oracle import forward as F
    n_layers = min(n_layers, cfg.n_layers)
    w = F.synth_weights(cfg, seed, fast=True, keep=True)
    a = F.synth_adapter(cfg, r, 1, fast=True) if r else None
    tok = synth.prompt_fast(cfg, S, 0)
    keep = tuple(f"model.layers.{i}." for i in range(n_layers))
    for s in synth.base_tensors(cfg):
        if not s.name.startswith("model.layers.") or s.name.startswith(keep):
            w(s.name)
    if a is not None:
        for s in synth.adapter_tensors(cfg, r):
            if s.name.startswith(keep):
                a(s.name)

    def run():
        t = time.perf_counter()
        F.forward(cfg, w, tok, a, 0x7F if r else 0, 1.0, n_layers=n_layers)
        return time.perf_counter() - t
    return run


def oracle_extrapolate(cfg, t_sample, n_layers=ORACLE_LAYERS):
    """Full-forward ms from a sample of n_layers (+ embed + head): layers
    scale linearly; the embed / head share is small (< 2 % at 13B)."""
    return t_sample * 1e3 * cfg.n_layers / min(n_layers, cfg.n_layers)


def workload_name(config, S, r):
    """The workload label both arms report (BASELINE.json configs[2] shape)."""
    return (f"Llama2-{config.upper()}-shaped prefill, S={S}, LoRA r{r} attach, template-start "
            f"(BASELINE.json configs[2])")


def run_reference(args):
    """--impl reference: the oracle (numpy fp32, plain definition) on the host
    cores, bounded samples of the same workload (1 of L layers, extrapolated)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.config(args.config)
    cores = len(os.sched_getaffinity(0))
    sample_fn = oracle_sampler(cfg, args.seq, args.rank)
    for _ in range(args.warmup):
        sample_fn()
    ts = [sample_fn() for _ in range(args.steps)]
    ms = oracle_extrapolate(cfg, statistics.median(ts))
    sample = (f"embed + {min(ORACLE_LAYERS, cfg.n_layers)} of {cfg.n_layers} layers + head at S={args.seq}, "
              f"r={args.rank}; value = median sample x {cfg.n_layers}/{min(ORACLE_LAYERS, cfg.n_layers)}")
    print(json.dumps({
        "impl": "reference", "metric": "template-start TTFT", "value": ms, "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # wall time of one timed step (one bounded sample), so steps x ms_per_step
        # matches the run's own clock; value extrapolates the sample to the workload
        "ms_per_step": statistics.mean(ts) * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded splitmix64 weights, uniform prompt)",
        "config": {"workload": workload_name(args.config, args.seq, args.rank),
                   "seq_len": args.seq, "lora_rank": args.rank,
                   "parallelism": f"tp{args.gpus}" if args.gpus > 1 else "single",
                   "reference": "oracle/ (numpy fp32 plain-definition forward) on the host "
                                "cores: the paper ships no code, so the oracle is this tier's "
                                "reference arm (DESIGN.md §10)"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def eq1_t_ttft(t_warm_s, adapter_bytes, b_pcie_Bps):
    """The T_TTFT handed to the planner's Eq. 1 (M_prefetch =
    max(M_model - T_TTFT x B_PCIe, 0)) so that it sizes the template for the
    invocation's whole footprint, base weights plus a dynamic adapter that
    always streams (reading A7b): M_model + M_adapter - T x B =
    M_model - (T - M_adapter / B) x B."""
    return max(t_warm_s - adapter_bytes / b_pcie_Bps, 0.0)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 outside torchrun: one rank per GPU via torch.distributed.run
    (127.0.0.1 rendezvous).  Fails loudly when fewer than N GPUs are visible:
    a silent world = 1 run would report n_gpus = 1 under an N-GPU request."""
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
                         f"found {n}; refusing to run a smaller world\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def h2d_bandwidth(torch, dist, nbytes=1 << 30, reps=10):
    """B_h2d(N) of SURVEY §8(d): per-GPU pinned->device copy of 1 GiB with all
    ranks copying at once (barrier before each rep), best of `reps`; bytes/s."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dv = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0.record()
        dv.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3))
    del h, dv
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tidal", choices=["tidal", "reference"])
    ap.add_argument("--config", default="13b")
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--rho", default="eq1")
    ap.add_argument("--eq1-adapter", default="on", choices=["on", "off"],
                    help="count the streamed adapter's bytes in Eq. 1 (reading A7b)")
    ap.add_argument("--policy", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--quick", action="store_true", help="profiling runs: minimal extra passes")
    ap.add_argument("--decode-steps", type=int, default=64,
                    help="greedy decode steps measured after the prefill (0: skip)")
    ap.add_argument("--allreduce", default="f32", choices=["f32", "bf16"],
                    help="TP row-parallel allreduce precision (N > 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        sys.stderr.write(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} GPU(s) visible\n")
        return 2
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2503_06421_b200 import build as B
    if rank == 0:
        synth.build_c() if not os.path.exists(os.path.join(ROOT, "synth", "libsynth.so")) else None
        B.build()
    if dist:
        dist.barrier()
    from paper_2503_06421_b200 import tidal as T

    cfg = synth.config(args.config)
    S, r = args.seq, args.rank
    P, peak_src = peaks()
    t_setup = time.perf_counter()
    tensors, fill = synth.model_inputs(cfg, 0, world, rank)
    model = T.Model(cfg_dict(cfg), tensors, "base:0", fill=fill, world=world, rank=rank)
    trace = T.Trace(model)     # planner trace == traced first run (tests/test_gpu_e2e.py)
    comm = None
    if world > 1:
        uid = [T.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = T.Comm(world, rank, uid[0], local)
    tpl = T.Template(model, trace, T.template_opts(resident_bytes=0, group_policy=args.policy,
                                                   max_tokens=S, device=local, comm=comm))
    abuf, anb, slots = None, 0, None
    if r:
        slots, anb = tpl.adapter_layout(r, 0x7F)
        abuf = T.PinnedBuffer(anb)
        synth.adapter_fill(cfg, r, 1, slots, abuf.view(), 0x7F, world, rank)
    tokens = synth.prompt_fast(cfg, S, 0)
    setup_s = time.perf_counter() - t_setup

    def attach():
        return T.Adapter(tpl, r, 1.0, 0x7F, abuf, anb, "adapter:1") if r else None

    def step(debug):
        tpl.set_debug(debug)
        h0 = time.perf_counter()
        ad = attach()
        attach_ms = (time.perf_counter() - h0) * 1e3
        tok, logits, st = tpl.invoke(tokens, ad)
        st["attach_ms"] = attach_ms
        st["e2e_ms"] = (time.perf_counter() - h0) * 1e3
        st["token"] = tok
        return st

    def reduce_ranks(x, op):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x):
        return reduce_ranks(x, dist.ReduceOp.MAX if dist else None)

    def min_over_ranks(x):
        return reduce_ranks(x, dist.ReduceOp.MIN if dist else None)

    def barrier():
        if dist:
            dist.barrier()

    if world > 1:
        tpl.set_allreduce_dtype(T.DTYPE_BF16 if args.allreduce == "bf16" else T.DTYPE_F32)
    # (0) B_h2d(N): raw 1 GiB pinned copies, all ranks at once
    b_raw_rank = h2d_bandwidth(torch, dist, reps=3 if args.quick else 10)
    b_raw = min_over_ranks(b_raw_rank)
    # (1) H2D bandwidth of this path and the load-then-infer baseline (rho = 0,
    # serial), every rank streaming its own shard at the same time
    for _ in range(1 if args.quick else 2):
        barrier()
        st0 = step(T.DEBUG_SERIAL | T.DEBUG_SCRUB_L2)
    h2d_ms = st0["h2d_last_ms"] - st0["h2d_first_ms"]
    stream_bytes = st0["bytes_streamed"] + st0["bytes_adapter"]
    b_h2d_rank = stream_bytes / (h2d_ms / 1e3)
    b_h2d = min_over_ranks(b_h2d_rank)   # the slowest link bounds a TP step
    cold_ms = max_over_ranks(st0["device_ms"])
    sweep = {"load_then_infer_rho0": cold_ms}
    if not args.no_sweep and not args.quick:
        barrier()
        sweep["overlap_rho0"] = max_over_ranks(step(T.DEBUG_SCRUB_L2)["device_ms"])
    # (2) warm TTFT (rho = 1), the T_TTFT of Eq. 1: same protocol as the timed
    # region (W warm-up + K back-to-back steps, L2 flushed, no profiling events)
    tpl.resize(T.template_opts(resident_bytes=T.U64_MAX))
    n_warm = 1 if args.quick else args.steps
    for _ in range(0 if args.quick else args.warmup):
        step(T.DEBUG_SCRUB_L2)
    barrier()
    warm = [step(T.DEBUG_SCRUB_L2)["device_ms"] for _ in range(n_warm)]
    t_warm = max_over_ranks(statistics.mean(warm))
    sweep["warm_rho1"] = t_warm
    tp_info = None
    if world > 1 and not args.quick:
        other = "bf16" if args.allreduce == "f32" else "f32"
        tpl.set_allreduce_dtype(T.DTYPE_BF16 if other == "bf16" else T.DTYPE_F32)
        step(T.DEBUG_SCRUB_L2)
        barrier()
        w2 = [step(T.DEBUG_SCRUB_L2)["device_ms"] for _ in range(n_warm)]
        sweep[f"warm_rho1_allreduce_{other}"] = max_over_ranks(statistics.mean(w2))
        tpl.set_allreduce_dtype(T.DTYPE_BF16 if args.allreduce == "bf16" else T.DTYPE_F32)
    # (3) template size
    # Eq. 1 balances loading against inference: every
    # invocation also streams its dynamic adapter (never template-resident),
    # so those bytes take their share of T_TTFT x B_PCIe and the template
    # absorbs it (reading A7b): M_prefetch = max(M_model +
    # M_adapter - T_TTFT x B_PCIe, 0), passed to the planner's Eq. 1 as
    # T' = T_TTFT - M_adapter / B_PCIe.  --eq1-adapter off: the adapter ignored.
    t_eq1 = eq1_t_ttft(t_warm / 1e3, anb if (args.eq1_adapter == "on" and r) else 0, b_h2d)
    if args.rho == "eq1":
        tpl.resize(T.template_opts(eq1=True, t_ttft_s=t_eq1, b_pcie_Bps=b_h2d))
    else:
        M = sum(s.nbytes for s in synth.base_tensors(cfg)) // world
        tpl.resize(T.template_opts(resident_bytes=int(float(args.rho) * M)))
    # (4) timed region: no events inside the forward (PDL overlap intact)
    dbg = T.DEBUG_SCRUB_L2
    for _ in range(args.warmup):
        step(dbg)
    barrier()
    torch.cuda.synchronize()
    stats = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            stats.append(step(dbg))
    torch.cuda.synchronize()
    barrier()
    # (5) the same K steps again with CUDA events around each tensor-core GEMM
    # (the dominant kernels): their per-launch time for `roofline`
    tpl.profile(reset=True)
    for _ in range(args.steps):
        step(T.DEBUG_SCRUB_L2 | T.DEBUG_PROFILE_GEMM)
    prof = tpl.profile(reset=True)
    # (6) per-kernel-class table: a separate pass with events around every launch
    # (bracketing adds a launch gap per kernel, so short kernels read high)
    n_all = 1 if args.quick else 3
    for _ in range(n_all):
        step(T.DEBUG_SCRUB_L2 | T.DEBUG_PROFILE)
    prof_all = tpl.profile(reset=True)
    if not args.quick and not args.no_sweep:
        # keep-alive with adapter hot-swap (Tidal-DK, §5.2): the streamed
        # weights of the previous invocation stay; only the adapter streams
        tpl.keep_alive()
        barrier()
        sweep["keep_alive_hot_swap"] = max_over_ranks(
            statistics.median(step(T.DEBUG_SCRUB_L2)["device_ms"] for _ in range(3)))
        # loading-order ablation at rho = 0 (§7.4)
        tpl.resize(T.template_opts(resident_bytes=0))
        for name, order in (("rho0_order_reverse", T.ORDER_REVERSE),
                            ("rho0_order_registration", T.ORDER_REGISTRATION)):
            tpl.set_load_order(order)
            barrier()
            sweep[name] = max_over_ranks(step(T.DEBUG_SCRUB_L2)["device_ms"])
        tpl.set_load_order(T.ORDER_TRACED)
    decode = None
    if world == 1 and not args.quick and args.decode_steps > 0:
        # decode continuation: greedy steps after the first
        # token, every weight read from HBM once per token; roofline = (weight
        # bytes + mean K/V bytes) / measured HBM bandwidth
        n = args.decode_steps
        tpl.enable_decode(n)
        per_tok = []
        for _ in range(3):
            tpl.set_debug(0)
            ad = attach()
            tpl.invoke(tokens, ad, want_logits=False)
            _, _, dst = tpl.decode(n, ad, want_logits=False)
            per_tok.append(dst["per_token_ms"])
        ms = statistics.median(per_tok)
        kv_mean = dst["kv_bytes_last_token"] * (S + n / 2) / (S + n)
        bytes_tok = dst["weight_bytes_per_token"] + kv_mean
        roof_ms = bytes_tok / (P["hbm_gbs"] * 1e9) * 1e3
        decode = {"steps": n, "after_prompt": S, "ms_per_token": ms, "tokens_per_s": 1e3 / ms,
                  "bytes_per_token": bytes_tok, "hbm_gbs_achieved": bytes_tok / (ms / 1e3) / 1e9,
                  "hbm_roof_ms_per_token": roof_ms, "frac": roof_ms / ms,
                  "kernels_per_token": dst["n_kernels"] / n,
                  "note": "CUDA-graph replay per token; weights resident after the prefill"}
    dev_ms = [max_over_ranks(s["device_ms"]) for s in stats]
    e2e_ms = [max_over_ranks(s["e2e_ms"]) for s in stats]
    s0 = stats[0]
    ttft = statistics.mean(dev_ms)
    if dist:
        # tear down in order on every rank (template before communicator before
        # the process group) so no rank exits through interpreter-shutdown GC
        dist.barrier()
        tpl = None
        comm = None
        dist.destroy_process_group()
    if rank != 0:
        return 0

    # roofline of the whole step (north_star): max(streamed / B_h2d, FLOPs / peak),
    # plus the HBM bound of reading every weight once (binds only for short prompts)
    flops = prefill_flops(cfg, S, r, world)
    streamed = s0["bytes_streamed"] + s0["bytes_adapter"]
    t_pcie = streamed / b_h2d * 1e3
    t_tc = flops / (P["bf16_tflops"] * 1e12) * 1e3
    w_bytes = s0["bytes_streamed"] + s0["bytes_resident"] + s0["bytes_adapter"]
    t_hbm = w_bytes / (P["hbm_gbs"] * 1e9) * 1e3
    roof = max(t_pcie, t_tc, t_hbm)
    bound = max((("pcie", t_pcie), ("tensor", t_tc), ("hbm", t_hbm)), key=lambda kv: kv[1])[0]
    # dominant kernel (largest device time in the timed region)
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = dom["ms"] / max(1, dom["launches"])
    tensor_bound = dom["flops"] > 0 and dom["flops"] / max(dom["bytes"], 1) > 50
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom_name)
        except Exception:
            traffic = None
    if tensor_bound:
        ach = dom["flops"] / (dom["ms"] / 1e3) / 1e12
        pk = P["bf16_tflops"]
        pks = P.get("bf16_tflops_sustained", pk)
        rl = {"kernel": dom_name, "bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
              "frac": ach / pk, "traffic": traffic, "frac_vs_sustained": ach / pks,
              "per_launch": {"ms": per_launch_ms, "flops": dom["flops"] / max(1, dom["launches"])},
              "timing": f"CUDA events around each launch on the compute stream, {args.steps} "
                        "steps after the timed region (same inputs, L2 flushed per step)",
              "peak_source": peak_src + " bf16_tflops (burst)"}
    else:
        ach = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
        rl = {"kernel": dom_name, "bound": "hbm", "achieved": ach, "peak": P["hbm_gbs"],
              "unit": "GB/s", "frac": ach / P["hbm_gbs"], "traffic": traffic,
              "per_launch": {"ms": per_launch_ms, "bytes": dom["bytes"] / max(1, dom["launches"])},
              "peak_source": peak_src}
    kernels = {k: {"ms_per_step": v["ms"] / n_all, "launches_per_step": v["launches"] / n_all,
                   "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None,
                   "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None}
               for k, v in prof_all.items() if v["launches"]}
    if world > 1:
        tot = sum(v["ms_per_step"] for v in kernels.values())
        ar = kernels.get("allreduce", {}).get("ms_per_step", 0.0)
        tp_info = {"allreduce_dtype": args.allreduce, "allreduce_ms_per_step": ar,
                   "allreduce_share": ar / tot if tot else None,
                   "note": "share of the all-kernel event pass (allreduce = NCCL on the "
                           "compute stream, incl. bf16 pack/add kernels when bf16)"}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample_fn = oracle_sampler(cfg, S, r)
        sample_fn()
        t1 = statistics.median(sample_fn() for _ in range(2))
        cpu = {"value": oracle_extrapolate(cfg, t1), "unit": "ms",
               "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"numpy fp32 oracle: embed + {ORACLE_LAYERS} of {cfg.n_layers} layers + "
                         f"head at S={S}, LoRA r{r}, median of 2 after 1 warm-up; "
                         f"value = t x {cfg.n_layers}/{min(ORACLE_LAYERS, cfg.n_layers)}",
               "sample_s": t1}
    out = {
        "metric": "template-start TTFT", "value": ttft, "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ttft,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded splitmix64 random-init bf16 weights + LoRA, uniform prompt)",
        "config": {"workload": workload_name(args.config, S, r),
                   "seq_len": S, "lora_rank": r, "resident_rule": (args.rho + ("+adapter" if args.eq1_adapter == "on" and r else ""))
                   if args.rho == "eq1" else args.rho,
                   "rho": s0["bytes_resident"] / max(1, s0["bytes_resident"] + s0["bytes_streamed"]),
                   "group_policy": args.policy, "parallelism": f"tp{world}" if world > 1 else "single",
                   "l2": "flushed before every step (512 MB write, outside the timed window)"},
        "ttft_ms": {"mean": ttft, "median": statistics.median(dev_ms),
                    "p95": sorted(dev_ms)[max(0, int(np.ceil(0.95 * len(dev_ms))) - 1)],
                    "min": min(dev_ms)},
        "tokens_per_s": S / (ttft / 1e3),
        "ttft_roofline": {"roof_ms": roof, "bound": bound,
                          "t_pcie_ms": t_pcie, "t_tensor_ms": t_tc, "t_hbm_ms": t_hbm,
                          "frac": roof / ttft,
                          "streamed_bytes_per_rank": streamed, "b_h2d_GBps": b_h2d / 1e9,
                          "b_h2d_this_rank_GBps": b_h2d_rank / 1e9,
                          "b_h2d_raw_GBps": b_raw / 1e9,
                          "b_h2d_note": "b_h2d: this path's own streaming rate in the serial rho=0 "
                                        "step, MIN over ranks, all ranks streaming at once; "
                                        "raw: 1 GiB pinned copy, best of 10, all ranks at once",
                          "flops_per_rank": flops, "peak_tflops": P["bf16_tflops"]},
        "roofline": rl,
        "cpu_baseline": cpu,
        "e2e": {"value": statistics.mean(e2e_ms), "unit": "ms",
                "h2d_bytes_per_step": int(4 * S + streamed),
                "d2h_bytes_per_step": int(4 * cfg.vocab + 8),
                "includes": "attach_lora + invoke (token H2D, weight/adapter H2D, logits D2H)"},
        "gpu_launches": int(sum(s["n_kernels"] for s in stats)),
        "kernels": kernels,
        "sweep_ms": sweep,
        "clocks": clk.summary(),
        "eq1": {"t_warm_ms": t_warm, "b_h2d_GBps": b_h2d / 1e9,
                "adapter_bytes_per_rank": anb if r else 0, "t_ttft_ms_passed": t_eq1 * 1e3,
                "adapter_counted": args.eq1_adapter == "on",
                "t_warm_protocol": f"mean of {n_warm} back-to-back rho=1 steps after "
                                   f"{args.warmup} warm-up, L2 flushed, no profiling events"},
        "tp": tp_info,
        # the compute-bound regime (fully template-resident, rho = 1): warm TTFT
        # against the tensor roof at the burst and at the sustained (power-cap)
        # measured bf16 peak; north_star's bar is frac >= 1/1.3
        "compute_bound_rho1": {
            "warm_ms": t_warm,
            "t_tensor_burst_ms": flops / (P["bf16_tflops"] * 1e12) * 1e3,
            "t_tensor_sustained_ms": flops / (P.get("bf16_tflops_sustained", P["bf16_tflops"]) * 1e12) * 1e3,
            "frac_burst": flops / (P["bf16_tflops"] * 1e12) * 1e3 / t_warm,
            "frac_sustained": flops / (P.get("bf16_tflops_sustained", P["bf16_tflops"]) * 1e12) * 1e3 / t_warm},
        "setup_s": setup_s,
        "first_token": s0["token"],
        "decode": decode,
    }
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main() or 0)
