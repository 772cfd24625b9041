"""Pins for oracle O2 (trace / template / fork plan) and O3 (overlap DES).

Fixed by: the SPEC.md worked examples (tests/golden/spec_examples.json), the
survey's hand-derived tiny plan (tests/golden/tiny_plan_r8_b50.txt), Table 1's
13B footprint ("24.3G" = 24.24 GiB), and invariants the paper
states (traced order beats init order, §7.4; overlap
bounds TTFT by max(load, compute), §5.2; barriers make every kernel
start after its weights land, line 555).
"""
import itertools
import json
import os
import random

import pytest

from oracle import des as D
from oracle import plan as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TINY = P.Shape(2, 256, 4, 4, 688, 1024)
B13 = P.Shape(40, 5120, 40, 40, 13824, 32000)
B7 = P.Shape(32, 4096, 32, 32, 11008, 32000)
B70 = P.Shape(80, 8192, 64, 8, 28672, 128256)


def _spec():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def _golden_lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.rstrip("\n") for l in f if l.strip() and not l.startswith("#")]


def test_tiny_worked_plan_matches_golden():
    tr = P.trace(TINY, "base:0")
    ad = P.adapter_tensors(TINY, 8, 0x7F, "adapter:0")
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=4213248 // 2), ad, 0x7F, 1, TINY)
    dump = P.plan_dump(p).splitlines()
    got = [l for l in dump if l.startswith(("GROUP", "BARRIER"))]
    assert got == _golden_lines("tiny_plan_r8_b50.txt")
    # resident = embed + all of layer 0 = 2,106,368 B (round-down tie-break)
    assert dump[-1] == "BYTES 2106368 2106880 156160 4213248"
    # R7 ACTION records against their hand derivation (VERDICT r1 weak #2c)
    assert [l for l in dump if l.startswith("ACTION")] == _golden_lines("tiny_actions_r8_b50.txt")


def test_tiny_layout_offsets():
    tr = P.trace(TINY, "base:0")
    p = P.make_plan(tr, P.TemplateOpts())
    assert p.offsets["model.embed_tokens.weight"] == 0
    assert p.offsets["model.layers.0.input_layernorm.weight"] == 524288
    assert p.offsets["model.layers.1.input_layernorm.weight"] == 2106368
    assert p.offsets["model.norm.weight"] == 3688448
    assert p.offsets["lm_head.weight"] == 3688960
    assert p.model_bytes == 4213248


def test_13b_footprint_matches_table1():
    tr = P.trace(B13, "base:0")
    M = sum(t.nbytes for t in tr.tensors)
    assert M == 26_031_728_640                    # 13,015,864,320 params x 2 B
    assert round(M / 2**30, 1) == 24.2            # Table 1 "24.3G" (GiB, rounding)
    assert abs(M / 2**30 - 24.3) < 0.1


def test_op_counts():
    for m in (TINY, B13, B70):
        assert len(P.op_sequence(m, 0, 1)) == 1 + 9 * m.n_layers + 3
        assert len(P.op_sequence(m, 0x7F, 8)) == 2 + 11 * m.n_layers + 4


def test_trace_first_read_semantics():
    ops = [("k0", ["w1"]), ("k1", ["w2"]), ("k2", ["w1"])]
    assert [n for n, _ in P.first_reads(ops)] == ["w1", "w2"]


def test_tied_embedding_accessed_first():
    m = P.Shape(2, 256, 4, 4, 688, 1024, tie_embeddings=True)
    tr = P.trace(m, "base:0")
    assert tr.access[0][0] == "model.embed_tokens.weight"
    assert "lm_head.weight" not in {t.name for t in tr.tensors}
    # lm_head op reads the alias; it collapses to the first read
    lm_op = [k for k, (o, _) in enumerate(tr.ops) if o == "lm_head"][0]
    assert tr.ops[lm_op][1] == ["model.embed_tokens.weight"]


def test_layout_is_permutation_and_r8_identity():
    rng = random.Random(0)
    for m in (TINY, B7, B13):
        tr = P.trace(m, "base:0")
        M = sum(t.nbytes for t in tr.tensors)
        for _ in range(20):
            budget = rng.randrange(0, M + 1)
            p = P.make_plan(tr, P.TemplateOpts(resident_bytes=budget))
            assert sorted(p.layout) == sorted(t.name for t in tr.tensors)
            res = sum(p.sizes[n] for n in p.layout[:p.n_resident])
            st = sum(p.sizes[n] for n in p.layout[p.n_resident:])
            assert res + st == M and res <= budget
            if p.n_resident < len(p.layout):
                assert res + p.sizes[p.layout[p.n_resident]] > budget


def test_eq1_examples_and_rounding():
    for ex in _spec()["eq1"]:
        assert P.eq1_prefetch_bytes(ex["model"], ex["t"], ex["b"]) == ex["expect"], ex["cite"]
    tr = P.trace(TINY, "base:0")
    sizes = [t.nbytes for t in tr.tensors]
    # round UP: smallest prefix covering M_pf
    k = P.resident_count([100, 200, 300], eq1_bytes=250)
    assert k == 2
    assert P.resident_count([100, 200, 300], eq1_bytes=0) == 0
    assert P.resident_count([100, 200, 300], budget=250) == 1


def test_eq1_monotone():
    rng = random.Random(1)
    for _ in range(1000):
        M = rng.randrange(0, 10**11)
        t, b = rng.uniform(0, 2), rng.uniform(1e9, 6e10)
        v = P.eq1_prefetch_bytes(M, t, b)
        assert 0 <= v <= M
        assert P.eq1_prefetch_bytes(M, t * 1.5, b) <= v
        assert P.eq1_prefetch_bytes(M, t, b * 1.5) <= v
        assert P.eq1_prefetch_bytes(M + 1000, t, b) >= v


def test_merge_examples():
    for ex in _spec()["merge"]:
        cuts = P.quantile_cuts([ex["size"]] * ex["n"], ex["G"])
        assert len(cuts) == ex["groups"], ex["cite"]
        assert all(len(c) == ex["per_group"] for c in cuts), ex["cite"]


def test_merge_properties():
    rng = random.Random(2)
    for _ in range(300):
        n = rng.randrange(1, 400)
        sizes = [rng.randrange(1, 10**6) for _ in range(n)]
        G = rng.randrange(1, 320)
        cuts = P.quantile_cuts(sizes, G)
        assert len(cuts) <= max(G, 1) or n <= G
        assert [i for c in cuts for i in c] == list(range(n))     # order-preserving partition


def test_per_tensor_and_max_transfers_policies():
    tr = P.trace(B70, "base:0", world=8)
    n = len(tr.tensors)
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=0, group_policy=P.POLICY_PER_TENSOR))
    assert len(p.groups) == n
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=0, group_policy=P.POLICY_MAX_TRANSFERS,
                                       max_transfers=300))
    assert len(p.groups) <= 300
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=0))
    assert len(p.groups) == 80 + 2


def test_barriers_cover_every_streamed_read():
    tr = P.trace(TINY, "base:0")
    ad = P.adapter_tensors(TINY, 8, 0x7F, "adapter:0")
    for budget in (0, 600000, 2106624, 4000000):
        for pol in (0, 1, 2):
            p = P.make_plan(tr, P.TemplateOpts(resident_bytes=budget, group_policy=pol,
                                               max_transfers=5), ad, 0x7F, 1, TINY)
            g_of = {n: g.idx for g in p.groups for n in g.members}
            for k, (_, reads) in enumerate(p.ops):
                need = {g_of[n] for n in reads if n in g_of}
                assert need == set(p.barriers.get(k, []))
            # resident weights are never in a group
            assert not set(p.layout[:p.n_resident]) & set(g_of)


def test_barrier_minimality_by_exhaustive_des():
    """Removing a group from the FIRST op that waits on it lets some copy order
    run that op before its weights land (SPEC.md fork-planner 'Minimality at
    group granularity'; later waits on the same group are implied by the
    in-order compute stream and are kept only as the R6 set definition)."""
    tr = P.trace(TINY, "base:0")
    ad = P.adapter_tensors(TINY, 8, 0x7F, "adapter:0")
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=600000), ad, 0x7F, 1, TINY)
    gb = [g.nbytes for g in p.groups]
    assert len(gb) <= 8
    dur = [1.0] * len(p.ops)
    first = {}
    for k in sorted(p.barriers):
        for g in p.barriers[k]:
            first.setdefault(g, k)
    assert sorted(first) == list(range(len(gb)))
    for g, k in first.items():
        if True:
            weak = {kk: [x for x in v if not (kk == k and x == g)] for kk, v in p.barriers.items()}
            violated = False
            for perm in itertools.permutations(range(len(gb))):
                sim = D.simulate(gb, 1e3, dur, weak, perm)
                if not D.residency_ok(sim, p.barriers):
                    violated = True
                    break
            assert violated, (k, g)
    # and with all barriers every order is safe
    for perm in itertools.permutations(range(len(gb))):
        assert D.residency_ok(D.simulate(gb, 1e3, dur, p.barriers, perm), p.barriers)


def test_cow_set_empty_for_forward():
    tr = P.trace(TINY, "base:0")
    p = P.make_plan(tr, P.TemplateOpts(resident_bytes=10**6))
    assert P.cow_set({}, p) == set()
    assert P.cow_set({3: ["model.layers.0.self_attn.q_proj.weight"]}, p) == \
        {"model.layers.0.self_attn.q_proj.weight"}
    assert P.cow_set({3: ["model.layers.0.self_attn.q_proj.lora_A"]}, p) == set()


def test_trace_dump_deterministic_and_complete():
    a = P.trace_dump(P.trace(TINY, "base:0"))
    b = P.trace_dump(P.trace(TINY, "base:0"))
    assert a == b
    lines = a.splitlines()
    assert sum(l.startswith("INIT") for l in lines) == 21
    assert sum(l.startswith("ACCESS") for l in lines) == 21
    assert lines[21] == "ACCESS 0 model.embed_tokens.weight embed#0"


def test_fnv1a64_known_vectors():
    # FNV-1a 64 published test vectors (offset basis for ""; "a")
    assert P.fnv1a64(b"") == 0xCBF29CE484222325
    assert P.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert P.fnv1a64(b"foobar") == 0x85944171F73967E8


# ---------------------------------------------------------------------------
# O3 DES
# ---------------------------------------------------------------------------
def test_des_spec_example():
    for ex in _spec()["des"]:
        bar = {int(k): v for k, v in ex["barriers"].items()}
        r = D.simulate(ex["bytes"], ex["bw"], ex["dur"], bar)
        assert r["op_end"] == ex["ends"] and r["ttft"] == ex["ttft"], ex["cite"]


def test_des_all_resident_is_sum():
    r = D.simulate([], 1.0, [0.5, 1.5, 2.0], {})
    assert r["ttft"] == 4.0


def test_des_overlap_bounds_and_traced_order_optimal():
    rng = random.Random(3)
    for _ in range(200):
        n = rng.randrange(1, 7)
        gb = [rng.uniform(0.1, 5) for _ in range(n)]
        dur = [rng.uniform(0.1, 3) for _ in range(n)]
        bar = {k: [k] for k in range(n)}          # single forward pass, op k reads group k
        r = D.simulate(gb, 2.0, dur, bar)
        copy = sum(gb) / 2.0
        assert max(sum(dur), copy) - 1e-9 <= r["ttft"] <= sum(dur) + copy + 1e-9
        best, _ = D.oracle_ttft(gb, 2.0, dur, bar)
        assert abs(best - r["ttft"]) < 1e-9


def test_des_traced_order_beats_init_order_tied_embedding():
    """PAPER.md §7.4 (lines 835-842): the shared embedding is initialised and
    loaded last but accessed first; loading in traced order wins."""
    gb = [2.0] + [1.0] * 5                        # embed + 5 layers, access order
    dur = [0.2] * 6
    bar = {k: [k] for k in range(6)}
    traced = D.simulate(gb, 1.0, dur, bar)["ttft"]
    init = D.simulate(gb, 1.0, dur, bar, [1, 2, 3, 4, 5, 0])["ttft"]
    rev = D.simulate(gb, 1.0, dur, bar, [5, 4, 3, 2, 1, 0])["ttft"]
    assert traced < init and traced < rev


def test_des_prefetch_monotone():
    tr = P.trace(TINY, "base:0")
    M = sum(t.nbytes for t in tr.tensors)
    prev = None
    for budget in range(0, M + 1, M // 20):
        p = P.make_plan(tr, P.TemplateOpts(resident_bytes=budget))
        gb = [g.nbytes for g in p.groups]
        r = D.simulate(gb, 1e6, [1e-3] * len(p.ops), p.barriers)["ttft"]
        if prev is not None:
            assert r <= prev + 1e-12
        prev = r
