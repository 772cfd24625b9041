"""Tensor-parallel dataflow on CPU with world_size 2 (gloo).

Mirrors, op for op, what run_forward does when world > 1 (
csrc/runtime.cu, csrc/nccl.cu): vocab-parallel embedding + allreduce (C3);
column-parallel q/k/v/gate/up with LoRA A whole and B row-sharded; local heads
with the GQA map; row-parallel o/down whose partial sums (rank 0 carries the
residual, other ranks start from zero) are allreduced (C1/C2), LoRA A
column-sharded / B whole (A14); vocab-parallel head with an allgather of the
logit slices and a max-reduce of the packed argmax key (C4).  Each rank builds
its shard with synth.shard_block — the same slicing bench.py feeds the library
— and rank 0 checks the result against the single-device oracle.
"""
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(spec, ns, seed, world, rank):
    r0, nr, c0, nc = synth.shard_block(spec, world, rank)
    full = synth.bf16_bits_to_f32(synth.tensor_bits(spec, ns, seed)).astype(np.float64)
    full = full.reshape(spec.shape if len(spec.shape) == 2 else (1, spec.shape[0]))
    out = full[r0:r0 + nr, c0:c0 + nc]
    return out.reshape(spec.shape) if len(spec.shape) == 1 else out


def _key(v, idx):
    u = int(np.array([v], np.float32).view(np.uint32)[0])
    u = (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)
    return (u << 32) | (0xFFFFFFFF - idx)


def _tp_forward(cfg, rank, world, tokens, r, mask, scale, allreduce, allgather):
    from oracle import forward as F
    base = {s.name: s for s in synth.base_tensors(cfg)}
    ads = {s.name: s for s in synth.adapter_tensors(cfg, r, mask)} if r else {}
    W = lambda n: _shard(base[n], synth.NS_BASE, 0, world, rank)
    A = lambda n: _shard(ads[n], synth.NS_ADAPTER, 1, world, rank)
    S, d, hd = len(tokens), cfg.d_model, cfg.head_dim
    H, KV = cfg.n_heads // world, cfg.n_kv_heads // world
    Vl = cfg.vocab // world
    eps = cfg.rms_eps

    def lin(x, layer, t):
        m = synth.module_name(layer, t)
        y = x @ W(m + ".weight").T
        if r and (mask >> synth.TARGETS.index(t)) & 1:
            y = y + scale * ((x @ A(m + ".lora_A").T) @ A(m + ".lora_B").T)
        return y

    E = W("model.embed_tokens.weight")
    X = np.zeros((S, d))
    mine = (tokens >= rank * Vl) & (tokens < (rank + 1) * Vl)
    X[mine] = E[tokens[mine] - rank * Vl]
    X = allreduce(X)                                          # embed_allreduce
    cos, sin = F.rope_cos_sin(S, hd, cfg.rope_theta, np.float64)
    for i in range(cfg.n_layers):
        p = f"model.layers.{i}."
        Xn = F.rmsnorm(X, W(p + "input_layernorm.weight"), eps)
        q = F.rope(lin(Xn, i, "q").reshape(S, H, hd), cos, sin)
        k = F.rope(lin(Xn, i, "k").reshape(S, KV, hd), cos, sin)
        v = lin(Xn, i, "v").reshape(S, KV, hd)
        O = F.causal_attention(q, k, v)
        X = allreduce((X if rank == 0 else 0 * X) + lin(O, i, "o"))      # attn_allreduce
        Hn = F.rmsnorm(X, W(p + "post_attention_layernorm.weight"), eps)
        h = F.silu(lin(Hn, i, "gate")) * lin(Hn, i, "up")
        X = allreduce((X if rank == 0 else 0 * X) + lin(h, i, "down"))   # mlp_allreduce
    hl = F.rmsnorm(X[-1:], W("model.norm.weight"), eps)[0]
    logits_r = W("lm_head.weight") @ hl
    logits = allgather(logits_r)                              # logits_allgather
    j = int(np.argmax(logits_r))
    key = allreduce(np.array([_key(float(logits_r[j]), rank * Vl + j)], dtype=np.uint64), op="max")
    return logits, 0xFFFFFFFF - (int(key[0]) & 0xFFFFFFFF)


def _worker(rank, world, port, cfg, r, mask, scale, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def allreduce(x, op="sum"):
            if x.dtype == np.uint64:        # gloo has no u64 max: gather and reduce
                g = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(g, torch.tensor(x.astype(np.int64)))
                return np.array([max(int(t.item()) & 0xFFFFFFFFFFFFFFFF for t in g)], np.uint64)
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        def allgather(x):
            g = [torch.zeros(len(x), dtype=torch.float64) for _ in range(world)]
            dist.all_gather(g, torch.from_numpy(np.ascontiguousarray(x)))
            return np.concatenate([t.numpy() for t in g])

        tokens = synth.prompt(cfg, 12, 3)
        logits, tok = _tp_forward(cfg, rank, world, tokens, r, mask, scale, allreduce, allgather)
        if rank == 0:
            q.put((logits, tok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,r,mask", [
    (synth.config("tiny"), 8, 0x7F),
    (synth.ModelConfig("gqa", 2, 256, 4, 2, 512, 512, rope_theta=500000.0), 16, 0x3B),
])
def test_tensor_parallel_dataflow_matches_oracle(cfg, r, mask):
    from oracle import forward as F
    mp = torch.multiprocessing.get_context("spawn")
    q = mp.Queue()
    port = _free_port()
    procs = [mp.Process(target=_worker, args=(k, 2, port, cfg, r, mask, 0.5, q)) for k in range(2)]
    for p in procs:
        p.start()
    logits, tok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tokens = synth.prompt(cfg, 12, 3)
    ref = F.forward(cfg, F.synth_weights(cfg, 0), tokens, F.synth_adapter(cfg, r, 1, mask), mask,
                    0.5, dtype=np.float64)
    assert np.abs(logits - ref["logits"]).max() < 1e-9
    assert tok == ref["token"]


def test_shards_tile_the_unsharded_tensor():
    cfg = synth.config("tiny")
    for spec in synth.base_tensors(cfg) + synth.adapter_tensors(cfg, 8):
        full = synth.tensor_bits(spec, 0, 0).reshape(spec.shape if len(spec.shape) == 2
                                                     else (1, spec.shape[0]))
        for world in (2, 4):
            cover = np.zeros(full.shape, dtype=int)
            for rk in range(world):
                r0, nr, c0, nc = synth.shard_block(spec, world, rk)
                cover[r0:r0 + nr, c0:c0 + nc] += 1
            replicated = len(spec.shape) == 1 or (cover == world).all()
            assert (cover == 1).all() or replicated, spec.name
