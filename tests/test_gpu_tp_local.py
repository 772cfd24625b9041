"""Tensor parallelism on one GPU: N in-process ranks (one thread each) share
cuda:0 through the local communicator (tidal_comm_create_local), so the whole
TP path — Megatron sharding of every weight and adapter (A14),
per-rank streaming, the C1/C2 allreduces, the vocab-parallel embed (C3) and
the argmax max-reduce + logits allgather (C4) — runs on the GPU against the
single-device oracle ("The TP oracle *is* the single-device
oracle").  Every rank must return the same token and bit-identical logits.
"""
import itertools
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import synth
from oracle import forward as F

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2
MARGIN = 2 * TOL
_uid = itertools.count()


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_06421_b200 import build
    build.build()
    from paper_2503_06421_b200 import tidal
    tidal.lib()
    return tidal


def cfg_dict(cfg):
    return dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
                n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
                rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps,
                tie_embeddings=cfg.tie_embeddings)


class Rank:
    def __init__(self, T, cfg, world, rank, group, rho, seed, policy):
        self.T, self.cfg, self.world, self.rank = T, cfg, world, rank
        tensors, fill = synth.model_inputs(cfg, seed, world, rank)
        self.model = T.Model(cfg_dict(cfg), tensors, f"base:{seed}", fill=fill, world=world, rank=rank)
        self.trace = T.Trace(self.model)
        self.comm = T.Comm(world, rank, device=0, local=group)
        M = sum(s.nbytes for s in synth.base_tensors(cfg)) // world
        self.tpl = T.Template(self.model, self.trace,
                              T.template_opts(resident_bytes=int(rho * M), group_policy=policy,
                                              max_tokens=512, device=0, comm=self.comm))

    def adapter(self, r, seed, mask, scale):
        slots, total = self.tpl.adapter_layout(r, mask)
        buf = self.T.PinnedBuffer(total)
        synth.adapter_fill(self.cfg, r, seed, slots, buf.view(), mask, self.world, self.rank)
        return self.T.Adapter(self.tpl, r, scale, mask, buf, total, f"adapter:{seed}")


def run_ranks(world, fn):
    with ThreadPoolExecutor(world) as ex:
        return list(ex.map(fn, range(world)))


def check_all(results, ref):
    tok0, l0, _ = results[0]
    for tok, logits, _ in results[1:]:
        assert tok == tok0 and np.array_equal(logits, l0)     # bit-identical on every rank
    err = float(np.abs(l0 - ref["logits"]).max())
    assert err <= TOL, err
    top = np.sort(ref["logits"])[-2:]
    if top[1] - top[0] > MARGIN:
        assert tok0 == ref["token"]
    assert ref["logits"][tok0] >= ref["logits"].max() - MARGIN
    return err


CASES = [
    # name, cfg, world, rho, policy, lora rank, mask, S
    ("tiny_tp2", synth.config("tiny"), 2, 0.5, 0, 8, 0x7F, 37),
    ("gqa128_tp2", synth.ModelConfig("gqa128", 2, 512, 4, 2, 1376, 2048, rope_theta=500000.0),
     2, 0.0, 0, 16, 0x7F, 300),
    ("hd128_tp4", synth.ModelConfig("hd128", 2, 1024, 8, 4, 2816, 4096), 4, 0.3, 2, 16, 0x35, 200),
    ("hd64_tp4_norank", synth.ModelConfig("hd64", 3, 512, 8, 4, 1408, 2048), 4, 1.0, 1, 0, 0, 129),
]


@pytest.mark.parametrize("name,cfg,world,rho,policy,r,mask,S", CASES, ids=[c[0] for c in CASES])
def test_tp_matches_single_device_oracle(T, name, cfg, world, rho, policy, r, mask, S):
    seed, aseed, scale = 7, 3, 0.75
    group = f"tp-{name}-{next(_uid)}"
    ranks = run_ranks(world, lambda k: Rank(T, cfg, world, k, group, rho, seed, policy))
    for rk in ranks:
        rk.tpl.set_debug(T.DEBUG_POISON)
    ads = [rk.adapter(r, aseed, mask, scale) if r else None for rk in ranks]
    tok = synth.prompt(cfg, S, 11)
    w = F.synth_weights(cfg, seed)
    ref = F.forward(cfg, w, tok, F.synth_adapter(cfg, r, aseed, mask) if r else None,
                    mask if r else 0, scale)
    c0 = [rk.tpl.checksum() for rk in ranks]
    for _ in range(2):
        res = run_ranks(world, lambda k: ranks[k].tpl.invoke(tok, ads[k]))
        check_all(res, ref)
    assert [rk.tpl.checksum() for rk in ranks] == c0
    # per-rank streaming: each rank moves only its own shard (plus its adapter slice)
    st = [x[2] for x in res]
    assert len({s["bytes_streamed"] + s["bytes_resident"] for s in st}) == 1


def test_tp_keep_alive_and_resize(T):
    cfg = synth.ModelConfig("gqa128", 2, 512, 4, 2, 1376, 2048, rope_theta=500000.0)
    world, seed = 2, 9
    group = f"tp-ka-{next(_uid)}"
    ranks = run_ranks(world, lambda k: Rank(T, cfg, world, k, group, 0.0, seed, 0))
    tok = synth.prompt(cfg, 64, 4)
    w = F.synth_weights(cfg, seed)
    a1 = [rk.adapter(8, 1, 0x7F, 1.0) for rk in ranks]
    check_all(run_ranks(world, lambda k: ranks[k].tpl.invoke(tok, a1[k])),
              F.forward(cfg, w, tok, F.synth_adapter(cfg, 8, 1), 0x7F, 1.0))
    for rk in ranks:
        rk.tpl.keep_alive()
    a2 = [rk.adapter(16, 2, 0x7F, 1.0) for rk in ranks]
    res = run_ranks(world, lambda k: ranks[k].tpl.invoke(tok, a2[k]))
    check_all(res, F.forward(cfg, w, tok, F.synth_adapter(cfg, 16, 2), 0x7F, 1.0))
    assert all(x[2]["bytes_streamed"] == 0 for x in res)
    run_ranks(world, lambda k: ranks[k].tpl.resize(T.template_opts(resident_bytes=T.U64_MAX, device=0,
                                                                   comm=ranks[k].comm)))
    check_all(run_ranks(world, lambda k: ranks[k].tpl.invoke(tok)), F.forward(cfg, w, tok))


def test_tp_batch(T):
    """Batched prompts under TP: logits come back [B][V] from the [world][B][V/world]
    device layout, per-prompt argmax max-reduced across ranks."""
    cfg = synth.ModelConfig("gqa128", 2, 512, 4, 2, 1376, 2048, rope_theta=500000.0)
    world, seed, B, Ls = 2, 12, 3, 150
    group = f"tp-batch-{next(_uid)}"
    ranks = run_ranks(world, lambda k: Rank(T, cfg, world, k, group, 0.3, seed, 0))
    ads = [rk.adapter(8, 4, 0x7F, 1.0) for rk in ranks]
    toks = np.stack([synth.prompt(cfg, Ls, 60 + b) for b in range(B)])
    res = run_ranks(world, lambda k: ranks[k].tpl.invoke_batch(toks, ads[k]))
    w = F.synth_weights(cfg, seed)
    aw = F.synth_adapter(cfg, 8, 4)
    for b in range(B):
        ref = F.forward(cfg, w, toks[b], aw, 0x7F, 1.0)
        check_all([(int(o[b]), l[b], s) for o, l, s in res], ref)
