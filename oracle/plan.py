"""O2 — trace, template and fork plan as text dumps (TEST INFRASTRUCTURE ONLY).

Follows the paper's pipeline in its own order:
  * lax inference tracing (§4.1: "capturing only the
    access patterns of weights, including their order and associated GPU
    kernels") -> ``trace``;
  * access-ordered layout and partial residency (§4.2: "reorganizes
    the weights based on the traced access order ... retains a subset of model
    weights on the GPU while preserving only the memory layouts of others");
  * template size by Eq. 1 (§5.2,
    M_prefetch = max(M_model - T_TTFT * B_PCIe, 0));
  * tensor merging into transfer groups (§6);
  * adaptive fork: resident weights reused by pointer, the rest loaded
    asynchronously in traced order, dynamic (adapter) weights re-initialised
    (§5.2), with sync events injected before each kernel that
    reads a not-yet-landed weight (line 555);
  * copy-on-write set = written ∩ forked (line 556) — empty for a forward.

The concrete rules R0-R8 (names, canonical op sequence, 256-B aligned layout,
round-down budget / round-up Eq. 1, per_layer / max_transfers / per_tensor
groups, barrier sets, dump grammar) are SURVEY.md §8(c) O2's readings of those
passages; DESIGN.md §Readings lists them.  The C-ABI planner must reproduce
these dumps byte for byte.  Pure Python, no numpy, no shared code.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

TARGETS = ("q", "k", "v", "o", "gate", "up", "down")
ALIGN = 256
POLICY_PER_LAYER, POLICY_MAX_TRANSFERS, POLICY_PER_TENSOR = 0, 1, 2
U64_MAX = (1 << 64) - 1


@dataclass(frozen=True)
class Shape:
    """Model shape (the fields of tidal_model_config)."""
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int
    vocab: int
    tie_embeddings: bool = False

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


@dataclass
class Tensor:
    name: str
    shape: Tuple[int, ...]
    kind: str            # "base" | "adapter"
    unit: int            # layer unit: 0 = embed, 1+i = layer i, L+1 = final
    provenance: str = ""

    @property
    def nbytes(self) -> int:
        n = 2
        for s in self.shape:
            n *= s
        return n


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & U64_MAX
    return h


def _mod(layer: int, t: str) -> str:
    return f"model.layers.{layer}.{'self_attn' if t in ('q', 'k', 'v', 'o') else 'mlp'}.{t}_proj"


# --------------------------------------------------------------------------
# R0 — names, registration order, rank-local shapes (TP: SURVEY.md §8(e), A14)
# --------------------------------------------------------------------------
def _proj_shape(m: Shape, t: str, world: int) -> Tuple[int, int]:
    hd = m.head_dim
    if t == "q":
        return (m.n_heads * hd // world, m.d_model)
    if t in ("k", "v"):
        return (m.n_kv_heads * hd // world, m.d_model)
    if t == "o":
        return (m.d_model, m.n_heads * hd // world)
    if t in ("gate", "up"):
        return (m.d_ff // world, m.d_model)
    return (m.d_model, m.d_ff // world)      # down


def _shape_str(shape: Sequence[int]) -> str:
    return "x".join(str(s) for s in shape)


def base_tensors(m: Shape, checkpoint: str, world: int = 1) -> List[Tensor]:
    """R0: HF state-dict order.  embed; per layer q,k,v,o,gate,up,down,
    input_layernorm, post_attention_layernorm; norm; lm_head (absent if tied)."""
    L = m.n_layers
    out = [Tensor("model.embed_tokens.weight", (m.vocab // world, m.d_model), "base", 0)]
    for i in range(L):
        for t in TARGETS:
            out.append(Tensor(_mod(i, t) + ".weight", _proj_shape(m, t, world), "base", 1 + i))
        out.append(Tensor(f"model.layers.{i}.input_layernorm.weight", (m.d_model,), "base", 1 + i))
        out.append(Tensor(f"model.layers.{i}.post_attention_layernorm.weight", (m.d_model,),
                          "base", 1 + i))
    out.append(Tensor("model.norm.weight", (m.d_model,), "base", L + 1))
    if not m.tie_embeddings:
        out.append(Tensor("lm_head.weight", (m.vocab // world, m.d_model), "base", L + 1))
    for t in out:
        t.provenance = f"{checkpoint}:{t.name}:{_shape_str(t.shape)}"
    return out


def adapter_tensors(m: Shape, rank: int, target_mask: int, checkpoint: str,
                    world: int = 1) -> List[Tensor]:
    """Adapter tensors in their own R0 order (per layer, per target: A then B).
    TP (A14): column-parallel targets keep A [r,in] whole and shard B rows;
    row-parallel targets (o, down) shard A columns and keep B [out,r] whole."""
    out = []
    for i in range(m.n_layers):
        for ti, t in enumerate(TARGETS):
            if not (target_mask >> ti) & 1:
                continue
            o, inn = _proj_shape(m, t, world)   # rank-local [out, in]
            out.append(Tensor(_mod(i, t) + ".lora_A", (rank, inn), "adapter", 1 + i))
            out.append(Tensor(_mod(i, t) + ".lora_B", (o, rank), "adapter", 1 + i))
    for t in out:
        t.provenance = f"{checkpoint}:{t.name}:{_shape_str(t.shape)}"
    return out


# --------------------------------------------------------------------------
# R1 — canonical logical-op sequence with read lists
# --------------------------------------------------------------------------
def op_sequence(m: Shape, target_mask: int = 0, world: int = 1) -> List[Tuple[str, List[str]]]:
    """[(op_name, reads)] in execution order.  LoRA entries only for attached
    targets (target_mask=0 -> no adapter).  world>1 inserts the TP exchange
    steps with empty read lists (embed_allreduce, attn/mlp_allreduce,
    logits_allgather)."""
    def lora(i: int, ts: Sequence[str]) -> List[str]:
        r = []
        for t in ts:
            if (target_mask >> TARGETS.index(t)) & 1:
                r += [_mod(i, t) + ".lora_A", _mod(i, t) + ".lora_B"]
        return r

    ops: List[Tuple[str, List[str]]] = [("embed", ["model.embed_tokens.weight"])]
    if world > 1:
        ops.append(("embed_allreduce", []))
    for i in range(m.n_layers):
        p = f"model.layers.{i}."
        ops.append(("attn_norm", [p + "input_layernorm.weight"]))
        ops.append(("qkv_proj", [_mod(i, t) + ".weight" for t in ("q", "k", "v")]
                    + lora(i, ("q", "k", "v"))))
        ops.append(("rope", []))
        ops.append(("attention", []))
        ops.append(("o_proj", [_mod(i, "o") + ".weight"] + lora(i, ("o",))))
        if world > 1:
            ops.append(("attn_allreduce", []))
        ops.append(("mlp_norm", [p + "post_attention_layernorm.weight"]))
        ops.append(("gate_up_proj", [_mod(i, "gate") + ".weight", _mod(i, "up") + ".weight"]
                    + lora(i, ("gate", "up"))))
        ops.append(("act_mul", []))
        ops.append(("down_proj", [_mod(i, "down") + ".weight"] + lora(i, ("down",))))
        if world > 1:
            ops.append(("mlp_allreduce", []))
    ops.append(("final_norm", ["model.norm.weight"]))
    ops.append(("lm_head", ["model.embed_tokens.weight" if m.tie_embeddings else "lm_head.weight"]))
    if world > 1:
        ops.append(("logits_allgather", []))
    ops.append(("argmax", []))
    return ops


def first_reads(ops: List[Tuple[str, List[str]]]) -> List[Tuple[str, int]]:
    """Access order = order of FIRST read (aliases collapse to the first read;
    SPEC.md tracer: "[w1],[w2],[w1] -> [w1, w2]").  Returns [(name, op_idx)]."""
    seen = set()
    order = []
    for k, (_, reads) in enumerate(ops):
        for n in reads:
            if n not in seen:
                seen.add(n)
                order.append((n, k))
    return order


# --------------------------------------------------------------------------
# Trace (tidal_trace) and its dump
# --------------------------------------------------------------------------
@dataclass
class Trace:
    tensors: List[Tensor]                 # registration order
    access: List[Tuple[str, int]]         # (name, op ordinal); never-read at tail (op -1)
    ops: List[Tuple[str, List[str]]]


def trace(m: Shape, checkpoint: str, world: int = 1) -> Trace:
    """Lax tracing of one first run with no adapter (§4.1)."""
    tensors = base_tensors(m, checkpoint, world)
    ops = op_sequence(m, 0, world)
    acc = first_reads(ops)
    seen = {n for n, _ in acc}
    names = {t.name for t in tensors}
    acc = [(n, k) for n, k in acc if n in names]
    acc += [(t.name, -1) for t in tensors if t.name not in seen]   # never-read tail
    return Trace(tensors, acc, ops)


def trace_dump(tr: Trace) -> str:
    lines = [f"INIT {t.name} {fnv1a64(t.provenance.encode()):016x} {t.nbytes}" for t in tr.tensors]
    for a, (n, k) in enumerate(tr.access):
        op = f"{tr.ops[k][0]}#{k}" if k >= 0 else "-"
        lines.append(f"ACCESS {a} {n} {op}")
    return "".join(l + "\n" for l in lines)


# --------------------------------------------------------------------------
# R3/R4 — layout and resident prefix (template), Eq. 1
# --------------------------------------------------------------------------
def align_up(x: int, a: int = ALIGN) -> int:
    return (x + a - 1) // a * a


def layout_offsets(sizes: Sequence[int]) -> Tuple[List[int], int]:
    """R3: running sum, each tensor start aligned to 256 B."""
    offs, cur = [], 0
    for s in sizes:
        cur = align_up(cur)
        offs.append(cur)
        cur += s
    return offs, cur


def eq1_prefetch_bytes(model_bytes: int, t_ttft_s: float, b_pcie_Bps: float) -> int:
    """Eq. 1: M_prefetch = max(M_model - T_TTFT*B_PCIe, 0).
    tb = floor(T*B) as one IEEE-double multiply, the rest integer (R4)."""
    tb = math.floor(t_ttft_s * b_pcie_Bps)
    return model_bytes - tb if model_bytes > tb else 0


def resident_count(sizes: Sequence[int], budget: Optional[int] = None,
                   eq1_bytes: Optional[int] = None) -> int:
    """R4: budget -> largest k with sum_{i<k} <= budget (round DOWN);
    Eq. 1 -> smallest k with sum_{i<k} >= M_prefetch (round UP)."""
    if eq1_bytes is not None:
        k, acc = 0, 0
        while acc < eq1_bytes and k < len(sizes):
            acc += sizes[k]
            k += 1
        return k
    if budget is None or budget >= U64_MAX:
        return len(sizes)
    k, acc = 0, 0
    while k < len(sizes) and acc + sizes[k] <= budget:
        acc += sizes[k]
        k += 1
    return k


@dataclass
class TemplateOpts:
    resident_bytes: int = U64_MAX
    eq1: bool = False
    t_ttft_s: float = 0.0
    b_pcie_Bps: float = 0.0
    group_policy: int = POLICY_PER_LAYER
    max_transfers: int = 300


@dataclass
class Group:
    idx: int
    kind: str              # base | adapter
    members: List[str]
    offset: int
    nbytes: int


@dataclass
class Plan:
    layout: List[str]                      # base layout (access order)
    offsets: Dict[str, int]
    n_resident: int
    adapter_layout: List[str]
    adapter_offsets: Dict[str, int]
    groups: List[Group]
    barriers: Dict[int, List[int]]
    sizes: Dict[str, int]
    model_bytes: int
    ops: List[Tuple[str, List[str]]]


# --------------------------------------------------------------------------
# R5 — transfer groups
# --------------------------------------------------------------------------
def quantile_cuts(sizes: Sequence[int], G: int) -> List[List[int]]:
    """max_transfers=G: one group per weight if n <= G (SPEC.md merge example
    "5 tensors, max 300 -> 5 singleton groups"); otherwise contiguous cuts at
    prefix-sum quantiles, exact integer arithmetic."""
    n = len(sizes)
    if n == 0:
        return []
    if n <= G:
        return [[i] for i in range(n)]
    total = sum(sizes)
    out, cur, k, cum = [], [], 1, 0
    for i, s in enumerate(sizes):
        cur.append(i)
        cum += s
        if cum * G >= k * total:
            out.append(cur)
            cur = []
            while k * total <= cum * G:
                k += 1
    if cur:
        out.append(cur)
    return out


def make_plan(tr: Trace, opts: TemplateOpts, adapter: Optional[List[Tensor]] = None,
              target_mask: int = 0, world: int = 1, m: Optional[Shape] = None) -> Plan:
    sizes = {t.name: t.nbytes for t in tr.tensors}
    units = {t.name: t.unit for t in tr.tensors}
    layout = [n for n, _ in tr.access]                        # base layout = access order
    lsizes = [sizes[n] for n in layout]
    offs, _ = layout_offsets(lsizes)
    model_bytes = sum(lsizes)
    if opts.eq1:
        k = resident_count(lsizes, eq1_bytes=eq1_prefetch_bytes(model_bytes, opts.t_ttft_s,
                                                                  opts.b_pcie_Bps))
    else:
        k = resident_count(lsizes, budget=opts.resident_bytes)

    adapter = adapter or []
    if adapter:
        assert m is not None
        ops = op_sequence(m, target_mask, world)
    else:
        ops = tr.ops
    for t in adapter:
        sizes[t.name] = t.nbytes
        units[t.name] = t.unit
    # combined first-read ordinals (base + adapter) for ordering groups
    acc_all = first_reads(ops)
    ordinal = {n: i for i, (n, _) in enumerate(acc_all)}
    a_names = {t.name for t in adapter}
    a_layout = [n for n, _ in acc_all if n in a_names]        # adapter access order
    a_offs, _ = layout_offsets([sizes[n] for n in a_layout])
    BIG = len(acc_all) + 10**9

    streamed = layout[k:]
    cand: List[Tuple[str, List[str]]] = []                    # (kind, members)
    if opts.group_policy == POLICY_PER_LAYER:
        by_unit: Dict[int, List[str]] = {}
        for n in streamed:
            by_unit.setdefault(units[n], []).append(n)
        for u in sorted(by_unit):
            cand.append(("base", by_unit[u]))
        a_by_unit: Dict[int, List[str]] = {}
        for n in a_layout:
            a_by_unit.setdefault(units[n], []).append(n)
        for u in sorted(a_by_unit):
            cand.append(("adapter", a_by_unit[u]))
    elif opts.group_policy == POLICY_MAX_TRANSFERS:
        for idxs in quantile_cuts([sizes[n] for n in streamed], opts.max_transfers):
            cand.append(("base", [streamed[i] for i in idxs]))
        for idxs in quantile_cuts([sizes[n] for n in a_layout], opts.max_transfers):
            cand.append(("adapter", [a_layout[i] for i in idxs]))
    else:
        cand += [("base", [n]) for n in streamed]
        cand += [("adapter", [n]) for n in a_layout]
    # groups ordered by the access ordinal of their first member
    cand.sort(key=lambda c: ordinal.get(c[1][0], BIG))

    base_off = dict(zip(layout, offs))
    ad_off = dict(zip(a_layout, a_offs))
    groups: List[Group] = []
    g_of: Dict[str, int] = {}
    for gi, (kind, mem) in enumerate(cand):
        o = base_off if kind == "base" else ad_off
        start = o[mem[0]]
        end = o[mem[-1]] + sizes[mem[-1]]
        groups.append(Group(gi, kind, mem, start, end - start))
        for n in mem:
            g_of[n] = gi
    # R6 barriers: set of groups holding any streamed/adapter weight op k reads
    barriers: Dict[int, List[int]] = {}
    for kk, (_, reads) in enumerate(ops):
        s = sorted({g_of[n] for n in reads if n in g_of})
        if s:
            barriers[kk] = s
    return Plan(layout, base_off, k, a_layout, ad_off, groups, barriers, sizes, model_bytes, ops)


def plan_dump(p: Plan) -> str:
    """R7 ACTION lines (layout order: RESIDENT, STREAM, then ADAPTER by group),
    R5 GROUP lines, R6 BARRIER lines, R8 BYTES accounting line."""
    lines = []
    for i, n in enumerate(p.layout):
        lines.append(f"ACTION {n} {'RESIDENT' if i < p.n_resident else 'STREAM'} {i}")
    a_index = {n: i for i, n in enumerate(p.adapter_layout)}
    for g in p.groups:
        if g.kind == "adapter":
            for n in g.members:
                lines.append(f"ACTION {n} ADAPTER {a_index[n]}")
    for g in p.groups:
        lines.append(f"GROUP {g.idx} {g.kind} {g.offset} {g.nbytes} {g.members[0]} {g.members[-1]}")
    for k in sorted(p.barriers):
        lines.append(f"BARRIER {k} {','.join(str(g) for g in p.barriers[k])}")
    res = sum(p.sizes[n] for n in p.layout[:p.n_resident])
    stream = sum(p.sizes[n] for n in p.layout[p.n_resident:])
    ad = sum(p.sizes[n] for n in p.adapter_layout)
    lines.append(f"BYTES {res} {stream} {ad} {p.model_bytes}")
    return "".join(l + "\n" for l in lines)


def cow_set(ops_writes: Dict[int, List[str]], p: Plan) -> set:
    """apply_cow (SPEC.md fork-planner): written ∩ (RESIDENT ∪ STREAM).
    Adapter weights are privately owned and never copied."""
    forked = set(p.layout)
    return {n for ws in ops_writes.values() for n in ws if n in forked}
