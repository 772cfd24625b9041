"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONE place both sides may import.  It holds no arithmetic of
the method (no norm, no GEMM, no attention, no plan rule): only the model
shapes of the paper's workloads and a counter-based generator for weights,
LoRA adapters and prompt tokens.  The paper (PAPER.md
§7.1) evaluates Llama-family checkpoints; there are no weights
on this box, so every tensor is drawn from splitmix64 with a variance-
preserving sigma (the paper is silent; DESIGN.md "Readings" R-init).

Two renderings exist and must be bit-identical (checked by a per-tensor hash
manifest in tests/test_synth.py):
  * ``synth`` (this file): numpy, the one the oracle tests use.
  * ``synth/csrc/synth.c`` -> ``synth/libsynth.so``: multithreaded C, used to
    fill the 13-26 GB pinned pools of the 7B/13B configs in seconds.

Generator:
  key  = splitmix64((ns << 56) ^ (seed << 24) ^ idx)
  u_e  = splitmix64(key + e)                     (e = row-major element index)
  x    = ((float)(u_e >> 40) * 2^-23 - 1) * c    (float32, one rounding)
  c    = (float)(sigma * sqrt(3))                (uniform with std sigma)
  w    = bf16_rne(x)            ; norm gains: bf16_rne(1.0f + x)
ns = 0 base weights, 1 adapter tensors, 2 prompt tokens.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, Tuple

import numpy as np

M64 = (1 << 64) - 1
NS_BASE, NS_ADAPTER, NS_TOKENS = 0, 1, 2

# LoRA target order (all 7 projections, Punica-style).
TARGETS = ("q", "k", "v", "o", "gate", "up", "down")


@dataclass(frozen=True)
class ModelConfig:
    """Llama-style decoder shape (BASELINE.json configs)."""
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    d_ff: int
    vocab: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    tie_embeddings: bool = False

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


# BASELINE.json configs[0..3].  tiny's F=688 is SURVEY.md §8(a)'s proposal.
CONFIGS: Dict[str, ModelConfig] = {
    "tiny": ModelConfig("tiny", 2, 256, 4, 4, 688, 1024),
    "7b": ModelConfig("7b", 32, 4096, 32, 32, 11008, 32000),
    "13b": ModelConfig("13b", 40, 5120, 40, 40, 13824, 32000),
    "70b": ModelConfig("70b", 80, 8192, 64, 8, 28672, 128256, rope_theta=500000.0),
}


def config(name: str, **over) -> ModelConfig:
    return replace(CONFIGS[name], **over) if over else CONFIGS[name]


# ----------------------------------------------------------------------------
# Tensor inventory of the synthetic checkpoint (HF state-dict names).  This is
# the *input* description (what the checkpoint contains and how each tensor is
# drawn); the oracle and the C++ planner each define their own registration /
# access order and are checked against one another, not against this list.
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: Tuple[int, ...]
    idx: int            # generator stream index (R0 registration index)
    sigma: float        # std of the uniform draw (double)
    is_norm: bool = False

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    @property
    def nbytes(self) -> int:
        return 2 * self.numel


def _proj_shapes(cfg: ModelConfig) -> Dict[str, Tuple[int, int]]:
    hd = cfg.head_dim
    d, F = cfg.d_model, cfg.d_ff
    return {
        "q": (cfg.n_heads * hd, d),
        "k": (cfg.n_kv_heads * hd, d),
        "v": (cfg.n_kv_heads * hd, d),
        "o": (d, cfg.n_heads * hd),
        "gate": (F, d),
        "up": (F, d),
        "down": (d, F),
    }


def _proj_sigma(cfg: ModelConfig, t: str) -> float:
    """Variance-preserving sigma (SURVEY.md §8(c) O0 'Proposed sigma')."""
    fan_in = _proj_shapes(cfg)[t][1]
    if t in ("o", "down"):
        return 1.0 / math.sqrt(float(fan_in) * 2 * cfg.n_layers)
    return 1.0 / math.sqrt(float(fan_in))


def module_name(layer: int, t: str) -> str:
    sub = "self_attn" if t in ("q", "k", "v", "o") else "mlp"
    return f"model.layers.{layer}.{sub}.{t}_proj"


def base_tensors(cfg: ModelConfig) -> List[TensorSpec]:
    """All base tensors with their generator index (registration order R0)."""
    out = [TensorSpec("model.embed_tokens.weight", (cfg.vocab, cfg.d_model), 0, 1.0)]
    shapes = _proj_shapes(cfg)
    for i in range(cfg.n_layers):
        base = 1 + 9 * i
        for j, t in enumerate(TARGETS):
            out.append(TensorSpec(module_name(i, t) + ".weight", shapes[t], base + j,
                                  _proj_sigma(cfg, t)))
        out.append(TensorSpec(f"model.layers.{i}.input_layernorm.weight", (cfg.d_model,),
                              base + 7, 0.05, True))
        out.append(TensorSpec(f"model.layers.{i}.post_attention_layernorm.weight",
                              (cfg.d_model,), base + 8, 0.05, True))
    out.append(TensorSpec("model.norm.weight", (cfg.d_model,), 1 + 9 * cfg.n_layers, 0.05, True))
    if not cfg.tie_embeddings:
        out.append(TensorSpec("lm_head.weight", (cfg.vocab, cfg.d_model), 2 + 9 * cfg.n_layers,
                              1.0 / math.sqrt(float(cfg.d_model))))
    return out


def adapter_tensors(cfg: ModelConfig, rank: int, target_mask: int = 0x7F) -> List[TensorSpec]:
    """LoRA A [r,in] / B [out,r] per targeted module.  Generator index is
    14*layer + 2*target + {0: A, 1: B} over ALL 7 targets, so a tensor's values
    do not depend on which other targets are attached (DESIGN.md reading)."""
    out = []
    shapes = _proj_shapes(cfg)
    for i in range(cfg.n_layers):
        for ti, t in enumerate(TARGETS):
            if not (target_mask >> ti) & 1:
                continue
            o, inn = shapes[t]
            sig_w = _proj_sigma(cfg, t)
            sa = 1.0 / math.sqrt(float(inn))
            sb = 0.25 * sig_w * math.sqrt(float(inn) / rank)
            out.append(TensorSpec(module_name(i, t) + ".lora_A", (rank, inn), 14 * i + 2 * ti, sa))
            out.append(TensorSpec(module_name(i, t) + ".lora_B", (o, rank), 14 * i + 2 * ti + 1, sb))
    return out


# ----------------------------------------------------------------------------
# splitmix64 and the element generator
# ----------------------------------------------------------------------------
def splitmix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_key(ns: int, seed: int, idx: int) -> int:
    assert 0 <= seed < (1 << 32) and 0 <= idx < (1 << 24)
    return splitmix64_int(((ns << 56) ^ (seed << 24) ^ idx) & M64)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (finite inputs)."""
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_bf16(ns: int, seed: int, idx: int, numel: int, sigma: float, is_norm: bool,
             start: int = 0) -> np.ndarray:
    """Elements [start, start+numel) of one tensor stream, as bf16 bits (uint16)."""
    key = stream_key(ns, seed, idx)
    e = np.arange(start, start + numel, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = _splitmix64_np(e + np.uint64(key))
    c = np.float32(sigma * math.sqrt(3.0))
    x = ((u >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)) * c
    if is_norm:
        x = np.float32(1.0) + x
    return f32_to_bf16_bits(x)


def tensor_bits(spec: TensorSpec, ns: int, seed: int) -> np.ndarray:
    return gen_bf16(ns, seed, spec.idx, spec.numel, spec.sigma, spec.is_norm).reshape(spec.shape)


def model_weights_bits(cfg: ModelConfig, seed: int) -> Dict[str, np.ndarray]:
    """name -> bf16 bits (uint16, HF shape).  numpy path: tiny / reduced configs."""
    return {s.name: tensor_bits(s, NS_BASE, seed) for s in base_tensors(cfg)}


def adapter_bits(cfg: ModelConfig, rank: int, seed: int, target_mask: int = 0x7F
                 ) -> Dict[str, np.ndarray]:
    return {s.name: tensor_bits(s, NS_ADAPTER, seed)
            for s in adapter_tensors(cfg, rank, target_mask)}


def prompt(cfg: ModelConfig, n_tokens: int, seed: int) -> np.ndarray:
    """tok_i = splitmix64(key(2, seed, 0) + i) mod V  (uniform ids; batch 1)."""
    key = stream_key(NS_TOKENS, seed, 0)
    e = np.arange(n_tokens, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = _splitmix64_np(e + np.uint64(key))
    return (u % np.uint64(cfg.vocab)).astype(np.int32)


def bits_hash(bits: np.ndarray) -> str:
    """Manifest hash of a bf16 tensor (little-endian bytes) for cross-checks."""
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(bits).astype("<u2").tobytes(),
                           digest_size=8).hexdigest()


# ----------------------------------------------------------------------------
# Fast path: the C rendering (synth/libsynth.so), same streams, many threads.
# ----------------------------------------------------------------------------
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        import ctypes
        import os
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "libsynth.so")
        if not os.path.exists(path):
            build_c()
        lib = ctypes.CDLL(path)
        lib.synth_fill_bf16.argtypes = [ctypes.c_uint64] * 3 + [ctypes.c_double, ctypes.c_int] + \
            [ctypes.c_uint64] * 5 + [ctypes.c_void_p, ctypes.c_int]
        lib.synth_fill_bf16.restype = ctypes.c_int
        lib.synth_prompt.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_void_p]
        _LIB = lib
    return _LIB


def build_c() -> str:
    import os
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    out = os.path.join(here, "libsynth.so")
    subprocess.check_call(["gcc", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                           os.path.join(here, "csrc", "synth.c"), "-o", out, "-lm"])
    return out


def n_threads() -> int:
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def fill_bf16(spec: TensorSpec, ns: int, seed: int, out_ptr: int, row0: int = 0,
              nrows: Optional[int] = None, col0: int = 0, ncols: Optional[int] = None,
              threads: Optional[int] = None) -> None:
    """C generator: write the [row0:row0+nrows, col0:col0+ncols] block of the
    unsharded tensor ``spec`` as bf16 bits to the raw pointer ``out_ptr``."""
    shape = spec.shape if len(spec.shape) == 2 else (1, spec.shape[0])
    nrows = shape[0] - row0 if nrows is None else nrows
    ncols = shape[1] - col0 if ncols is None else ncols
    _lib().synth_fill_bf16(ns, seed, spec.idx, spec.sigma, int(spec.is_norm), shape[1], row0,
                           nrows, col0, ncols, out_ptr, threads or n_threads())


def tensor_bits_fast(spec: TensorSpec, ns: int, seed: int) -> np.ndarray:
    out = np.empty(spec.shape, dtype=np.uint16)
    fill_bf16(spec, ns, seed, out.ctypes.data)
    return out


def prompt_fast(cfg: ModelConfig, n_tokens: int, seed: int) -> np.ndarray:
    out = np.empty(n_tokens, dtype=np.int32)
    _lib().synth_prompt(seed, cfg.vocab, n_tokens, out.ctypes.data)
    return out


# ----------------------------------------------------------------------------
# Tensor-parallel shards: every shard is a slice of the
# UNSHARDED tensor, so the weights are identical at every world size.
#   column-parallel (rows split): q, k, v, gate, up, embed, lm_head
#   row-parallel (columns split): o, down;   norms replicated
#   adapters (A14): q/k/v/gate/up -> A whole, B rows split;
#                   o/down        -> A columns split, B whole
# ----------------------------------------------------------------------------
def _target_of(name: str) -> Optional[str]:
    for t in TARGETS:
        if f".{t}_proj." in name:
            return t
    return None


def shard_block(spec: TensorSpec, world: int, rank: int) -> Tuple[int, int, int, int]:
    """(row0, nrows, col0, ncols) of this rank's slice of ``spec``."""
    if len(spec.shape) == 1:
        return 0, 1, 0, spec.shape[0]
    R, Cc = spec.shape
    if world == 1:
        return 0, R, 0, Cc
    t = _target_of(spec.name)
    is_a, is_b = spec.name.endswith("lora_A"), spec.name.endswith("lora_B")
    if t in ("o", "down"):
        if is_b:
            return 0, R, 0, Cc
        return 0, R, rank * Cc // world, Cc // world           # W [d, in] / A [r, in]
    if is_a:
        return 0, R, 0, Cc                                       # column-parallel A whole
    return rank * R // world, R // world, 0, Cc                  # W / B / embed / head rows


def model_inputs(cfg: ModelConfig, seed: int, world: int = 1, rank: int = 0):
    """[(name, nbytes, None)] + fill(dst, nbytes, index) for a tidal_model whose
    tensors are generated straight into the library's pinned pool."""
    specs = base_tensors(cfg)
    blocks = [shard_block(s, world, rank) for s in specs]
    tensors = [(s.name, 2 * b[1] * b[3], None) for s, b in zip(specs, blocks)]

    def fill(dst: int, nbytes: int, index: int) -> None:
        s, (r0, nr, c0, nc) = specs[index], blocks[index]
        assert nbytes == 2 * nr * nc
        fill_bf16(s, NS_BASE, seed, dst, row0=r0, nrows=nr, col0=c0, ncols=nc)
    return tensors, fill


def adapter_fill(cfg: ModelConfig, rank: int, seed: int, slots, buf: np.ndarray,
                 target_mask: int = 0x7F, world: int = 1, tp_rank: int = 0) -> None:
    """Write the seeded adapter into ``buf`` (uint8 view of a pinned buffer)
    at the canonical slots returned by tidal_adapter_layout."""
    specs = {s.name: s for s in adapter_tensors(cfg, rank, target_mask)}
    base = buf.ctypes.data
    for sl in slots:
        s = specs[sl["name"]]
        r0, nr, c0, nc = shard_block(s, world, tp_rank)
        assert sl["bytes"] == 2 * nr * nc, sl
        fill_bf16(s, NS_ADAPTER, seed, base + sl["offset"], row0=r0, nrows=nr, col0=c0, ncols=nc)
