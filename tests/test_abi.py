"""C-ABI on a CPU-only box: libtidal.so loads, exports every symbol declared in
include/*.h, and its planner (DRY mode, device = -1) reproduces the oracle's
trace and plan dumps byte for byte ("the load plan and trace
order bit-exact").  No compute calls are made here."""
import os
import random
import re
import subprocess

import pytest

import synth
from oracle import plan as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    from paper_2503_06421_b200 import build
    build.build()
    from paper_2503_06421_b200 import tidal
    tidal.lib()
    return tidal


def _declared_symbols():
    names = set()
    for h in ("tidal.h", "tidal_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(tidal_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(T):
    declared = _declared_symbols()
    assert len(declared) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", T.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = declared - exported
    assert not missing, missing
    bound = {n for n, _, _ in T.SIGNATURES}
    assert declared <= bound | {"tidal_trace"}, declared - bound


def test_library_is_sm100a_tcgen05(T):
    sass = subprocess.run(["cuobjdump", "-sass", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass          # tcgen05.mma + TMA
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", T.LIB_PATH], capture_output=True,
                                       text=True).stdout


def _cfg_dict(cfg):
    return dict(n_layers=cfg.n_layers, d_model=cfg.d_model, n_heads=cfg.n_heads,
                n_kv_heads=cfg.n_kv_heads, d_ff=cfg.d_ff, vocab=cfg.vocab,
                rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps,
                tie_embeddings=cfg.tie_embeddings)


def _shape(cfg):
    return P.Shape(cfg.n_layers, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.d_ff, cfg.vocab,
                   cfg.tie_embeddings)


def _dry(T, cfg, world=1, rank=0, ckpt="base:0"):
    tensors, fill = synth.model_inputs(cfg, 0, world, rank)
    m = T.Model(_cfg_dict(cfg), tensors, ckpt, fill=lambda *a: None, world=world, rank=rank)
    return m, T.Trace(m)


CASES = [("tiny", 1, 0), ("7b", 1, 0), ("13b", 1, 0), ("70b", 8, 3), ("13b", 2, 1)]


@pytest.mark.parametrize("name,world,rank", CASES)
def test_trace_dump_matches_oracle(T, name, world, rank):
    cfg = synth.config(name)
    _, tr = _dry(T, cfg, world, rank)
    assert tr.dump() == P.trace_dump(P.trace(_shape(cfg), "base:0", world))


def test_trace_dump_tied(T):
    cfg = synth.config("tiny", tie_embeddings=True)
    _, tr = _dry(T, cfg)
    assert tr.dump() == P.trace_dump(P.trace(_shape(cfg), "base:0"))


def _adapter_plan(T, tpl, cfg, rank, mask, world=1):
    slots, total = tpl.adapter_layout(rank, mask)
    a = T.Adapter(tpl, rank, 1.0, mask, None, total, "adapter:5")
    ad = P.adapter_tensors(_shape(cfg), rank, mask, "adapter:5", world)
    return a, ad, slots, total


@pytest.mark.parametrize("name,world,rank", CASES)
def test_plan_dump_matches_oracle(T, name, world, rank):
    cfg = synth.config(name)
    shape = _shape(cfg)
    m, tr = _dry(T, cfg, world, rank)
    otr = P.trace(shape, "base:0", world)
    M = sum(t.nbytes for t in otr.tensors)
    rng = random.Random(hash((name, world)) & 0xFFFF)
    budgets = [0, M // 2, M, P.U64_MAX] + [rng.randrange(0, M) for _ in range(3)]
    for budget in budgets:
        for pol in (0, 1, 2):
            opts = T.template_opts(resident_bytes=budget, group_policy=pol, max_transfers=37)
            tpl = T.Template(m, tr, opts)
            o = P.make_plan(otr, P.TemplateOpts(resident_bytes=budget, group_policy=pol,
                                                max_transfers=37))
            assert tpl.plan_dump() == P.plan_dump(o), (budget, pol)
            for r, mask in ((16, 0x7F), (8, 0x0F)):
                a, ad, _, _ = _adapter_plan(T, tpl, cfg, r, mask, world)
                o = P.make_plan(otr, P.TemplateOpts(resident_bytes=budget, group_policy=pol,
                                                    max_transfers=37), ad, mask, world, shape)
                assert tpl.plan_dump(a) == P.plan_dump(o), (budget, pol, r, mask)


def test_eq1_plan_and_resize_match_oracle(T):
    cfg = synth.config("13b")
    shape = _shape(cfg)
    m, tr = _dry(T, cfg)
    otr = P.trace(shape, "base:0")
    tpl = T.Template(m, tr, T.template_opts(resident_bytes=0))
    for t_s, bw in ((0.0318, 55.3e9), (0.3, 32e9), (1.0, 60e9), (0.0, 1.0)):
        tpl.resize(T.template_opts(eq1=True, t_ttft_s=t_s, b_pcie_Bps=bw))
        o = P.make_plan(otr, P.TemplateOpts(eq1=True, t_ttft_s=t_s, b_pcie_Bps=bw))
        assert tpl.plan_dump() == P.plan_dump(o)
        a, ad, _, _ = _adapter_plan(T, tpl, cfg, 16, 0x7F)
        o = P.make_plan(otr, P.TemplateOpts(eq1=True, t_ttft_s=t_s, b_pcie_Bps=bw), ad, 0x7F, 1,
                        shape)
        assert tpl.plan_dump(a) == P.plan_dump(o)


def test_tiny_plan_golden_via_abi(T):
    cfg = synth.config("tiny")
    m, tr = _dry(T, cfg, ckpt="base:0")
    tpl = T.Template(m, tr, T.template_opts(resident_bytes=4213248 // 2))
    a, _, slots, total = _adapter_plan(T, tpl, cfg, 8, 0x7F)
    assert total == 156160
    gold = [l.rstrip("\n") for l in open(os.path.join(ROOT, "tests/golden/tiny_plan_r8_b50.txt"))
            if l.strip() and not l.startswith("#")]
    got = [l for l in tpl.plan_dump(a).splitlines() if l.startswith(("GROUP", "BARRIER"))]
    assert got == gold


def test_structure_errors(T):
    cfg = synth.config("tiny")
    tensors, fill = synth.model_inputs(cfg, 0)
    with pytest.raises(T.TidalError) as e:
        T.Model(_cfg_dict(cfg), tensors[:-1], fill=fill)
    assert e.value.code == 5
    bad = list(tensors)
    bad[3] = (bad[3][0], bad[3][1] + 2, None)
    with pytest.raises(T.TidalError) as e:
        T.Model(_cfg_dict(cfg), bad, fill=fill)
    assert e.value.code == 5
    m, tr = _dry(T, cfg)
    tpl = T.Template(m, tr, T.template_opts())
    with pytest.raises(T.TidalError) as e:
        T.Adapter(tpl, 12, 1.0, 0x7F, None, 100)
    assert e.value.code == 1
    slots, total = tpl.adapter_layout(16)
    with pytest.raises(T.TidalError) as e:
        T.Adapter(tpl, 16, 1.0, 0x7F, None, total + 256)
    assert e.value.code == 5
    with pytest.raises(T.TidalError) as e:                 # dry template cannot run
        tpl.invoke(synth.prompt(cfg, 4, 0))
    assert e.value.code == 1


def test_adapter_layout_slots_cover_buffer(T):
    cfg = synth.config("tiny")
    m, tr = _dry(T, cfg)
    tpl = T.Template(m, tr, T.template_opts())
    slots, total = tpl.adapter_layout(8, 0x7F)
    assert len(slots) == 28
    end = 0
    for s in slots:
        assert s["offset"] % 256 == 0 and s["offset"] >= end
        end = s["offset"] + s["bytes"]
    assert end == total
    # order = adapter access order: q.A, q.B, k.A, ... (qkv_proj reads)
    assert slots[0]["name"].endswith("q_proj.lora_A") and slots[1]["name"].endswith("q_proj.lora_B")
