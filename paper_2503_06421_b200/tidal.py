"""Thin ctypes binding of libtidal.so (include/tidal.h, include/tidal_kernels.h).

Argument marshalling only: every step of the path runs in the library's
sm_100a kernels.  If the shared library is missing this module raises at
import time — there is no CPU fallback.  Names mirror the C-ABI.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtidal.so")

OK = 0
ERR_INVALID, ERR_STRUCTURE, ERR_BUFSZ = 1, 5, 8
ERR_NAMES = {0: "OK", 1: "INVALID", 2: "OOM", 3: "CUDA", 4: "NCCL", 5: "STRUCTURE",
             6: "RESIDENCY", 7: "COW", 8: "BUFSZ", 9: "NUMERIC"}
GROUPS_PER_LAYER, GROUPS_MAX_TRANSFERS, GROUPS_PER_TENSOR = 0, 1, 2
DEBUG_POISON, DEBUG_SKIP_BARRIER, DEBUG_SCRUB_L2, DEBUG_SERIAL, DEBUG_PROFILE = 1, 2, 4, 8, 16
DEBUG_PROFILE_GEMM = 32
DEBUG_NO_GRAPH = 64
DEBUG_TIMELINE = 128
ORDER_TRACED, ORDER_REVERSE, ORDER_REGISTRATION = 0, 1, 2
DTYPE_F32, DTYPE_BF16 = 0, 1
U64_MAX = (1 << 64) - 1


class TidalError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tidal {ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


class ModelConfig(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d_model", C.c_int), ("n_heads", C.c_int),
                ("n_kv_heads", C.c_int), ("d_ff", C.c_int), ("vocab", C.c_int),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("tie_embeddings", C.c_int)]


class HostTensor(C.Structure):
    _fields_ = [("name", C.c_char_p), ("host_bf16", C.c_void_p), ("bytes", C.c_size_t)]


class TemplateOpts(C.Structure):
    _fields_ = [("resident_bytes", C.c_uint64), ("eq1", C.c_int), ("t_ttft_s", C.c_double),
                ("b_pcie_Bps", C.c_double), ("group_policy", C.c_int),
                ("max_transfers", C.c_int), ("max_tokens", C.c_int), ("device", C.c_int),
                ("comm", C.c_void_p)]


class Slot(C.Structure):
    _fields_ = [("name", C.c_char_p), ("offset", C.c_uint64), ("bytes", C.c_uint64),
                ("rows", C.c_int), ("cols", C.c_int)]


class LoraDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("scale", C.c_float), ("target_mask", C.c_uint32),
                ("host_pinned", C.c_void_p), ("bytes", C.c_uint64), ("checkpoint", C.c_char_p)]


class Stats(C.Structure):
    _fields_ = [("ttft_host_ms", C.c_double), ("device_ms", C.c_double),
                ("h2d_first_ms", C.c_double), ("h2d_last_ms", C.c_double),
                ("compute_first_ms", C.c_double), ("compute_last_ms", C.c_double),
                ("bytes_streamed", C.c_uint64), ("bytes_resident", C.c_uint64),
                ("bytes_adapter", C.c_uint64), ("n_copies", C.c_int), ("n_kernels", C.c_int)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class DecodeStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("per_token_ms", C.c_double),
                ("weight_bytes_per_token", C.c_uint64), ("kv_bytes_last_token", C.c_uint64),
                ("n_kernels", C.c_int)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char_p), ("total_ms", C.c_double), ("launches", C.c_long),
                ("flops", C.c_double), ("bytes", C.c_double)]


FILL_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_void_p)
VP = C.c_void_p

# (name, restype, argtypes) of every exported symbol declared in include/*.h
SIGNATURES = [
    ("tidal_last_error", C.c_char_p, []),
    ("tidal_version", C.c_char_p, []),
    ("tidal_model_create", C.c_int, [C.POINTER(ModelConfig), C.POINTER(HostTensor), C.c_int,
                                     C.c_char_p, FILL_FN, VP, C.c_int, C.c_int, C.POINTER(VP)]),
    ("tidal_model_destroy", None, [VP]),
    ("tidal_trace", C.c_int, [VP, VP, C.c_int, C.c_int, VP, VP, VP, C.POINTER(VP)]),
    ("tidal_trace_destroy", None, [VP]),
    ("tidal_trace_dump", C.c_int, [VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("tidal_template_create", C.c_int, [VP, VP, C.POINTER(TemplateOpts), C.POINTER(VP)]),
    ("tidal_template_export", C.c_int, [VP, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("tidal_template_import", C.c_int, [VP, VP, C.POINTER(TemplateOpts), C.POINTER(C.c_int),
                                        C.c_int, C.c_uint64, C.c_uint64, C.POINTER(VP)]),
    ("tidal_template_resize", C.c_int, [VP, C.POINTER(TemplateOpts)]),
    ("tidal_template_keep_alive", C.c_int, [VP]),
    ("tidal_set_load_order", C.c_int, [VP, C.c_int]),
    ("tidal_template_destroy", None, [VP]),
    ("tidal_adapter_layout", C.c_int, [VP, C.c_int, C.c_uint32, C.POINTER(Slot), C.c_int,
                                       C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    ("tidal_attach_lora", C.c_int, [VP, C.POINTER(LoraDesc), C.POINTER(VP)]),
    ("tidal_adapter_destroy", None, [VP]),
    ("tidal_plan_dump", C.c_int, [VP, VP, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("tidal_invoke_prefill", C.c_int, [VP, VP, VP, C.c_int, VP, VP, C.POINTER(Stats)]),
    ("tidal_template_enable_decode", C.c_int, [VP, C.c_int]),
    ("tidal_invoke_decode", C.c_int, [VP, VP, C.c_int, VP, VP, C.POINTER(DecodeStats)]),
    ("tidal_invoke_prefill_batch", C.c_int,
     [VP, VP, VP, C.c_int, C.c_int, VP, VP, C.POINTER(Stats)]),
    ("tidal_set_device_allocator", C.c_int, [ALLOC_FN, FREE_FN, VP]),
    ("tidal_host_alloc", C.c_int, [C.c_uint64, C.POINTER(VP)]),
    ("tidal_host_free", None, [VP]),
    ("tidal_comm_unique_id", C.c_int, [VP]),
    ("tidal_comm_create", C.c_int, [C.c_int, C.c_int, VP, C.c_int, C.POINTER(VP)]),
    ("tidal_comm_create_local", C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_int, C.POINTER(VP)]),
    ("tidal_comm_destroy", None, [VP]),
    ("tidal_comm_selftest", C.c_int, [VP, C.c_uint64]),
    ("tidal_set_debug", C.c_int, [VP, C.c_int, C.c_int]),
    ("tidal_set_allreduce_dtype", C.c_int, [VP, C.c_int]),
    ("tidal_timeline_read", C.c_int, [VP, VP, C.c_int, VP, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    ("tidal_template_checksum", C.c_int, [VP, C.POINTER(C.c_uint64)]),
    ("tidal_profile_read", C.c_int, [VP, C.POINTER(KernelTime), C.c_int, C.POINTER(C.c_int),
                                     C.c_int]),
    ("tidal_weight_ptr", C.c_int, [VP, C.c_char_p, C.POINTER(VP)]),
    ("tidal_k_rmsnorm", C.c_int, [VP, VP, VP, C.c_int, C.c_int, C.c_float]),
    ("tidal_k_embed", C.c_int, [VP, VP, VP, C.c_int, C.c_int, C.c_int, C.c_int]),
    ("tidal_k_lora_shrink", C.c_int, [VP, C.c_int, C.c_int, VP, VP, C.c_int, C.c_float]),
    ("tidal_k_attention", C.c_int, [VP, VP, C.c_int, C.c_int, C.c_int, C.c_int]),
    ("tidal_k_head", C.c_int, [VP, VP, VP, C.c_int, C.c_int, C.c_float, VP, VP]),
    ("tidal_k_attention_tc", C.c_int, [VP, VP, C.c_int, VP, C.c_int, C.c_int, C.c_int]),
    ("tidal_k_gemm", C.c_int, [C.c_int, VP, C.POINTER(VP), C.POINTER(C.c_int), C.c_int, VP,
                               C.c_int, C.c_int, C.c_int, C.POINTER(VP), C.POINTER(VP), C.c_int,
                               VP, C.c_int]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libtidal.so; raise loudly if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2503_06421_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != OK:
        raise TidalError(rc, lib().tidal_last_error().decode())


def _dump(fn, *args) -> str:
    need = C.c_size_t(0)
    _check(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(fn(*args, buf, need.value, C.byref(need)))
    return buf.value.decode()


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()          # torch tensor (device memory)


# ---------------------------------------------------------------------------
class Model:
    """tidal_model: tensors given as (name, nbytes, host array or None); a
    ``fill(dst_ptr, nbytes, index)`` callable produces tensors without data."""

    def __init__(self, cfg: dict, tensors: Sequence[Tuple[str, int, Optional[np.ndarray]]],
                 checkpoint: str = "base", fill: Optional[Callable[[int, int, int], None]] = None,
                 world: int = 1, rank: int = 0):
        self._cfg = ModelConfig(cfg["n_layers"], cfg["d_model"], cfg["n_heads"],
                                cfg["n_kv_heads"], cfg["d_ff"], cfg["vocab"],
                                cfg.get("rope_theta", 1e4), cfg.get("rms_eps", 1e-5),
                                int(cfg.get("tie_embeddings", False)))
        self.vocab = cfg["vocab"]
        self._keep = [a for _, _, a in tensors if a is not None]
        arr = (HostTensor * len(tensors))()
        self._names = [n.encode() for n, _, _ in tensors]
        for i, (n, b, a) in enumerate(tensors):
            arr[i] = HostTensor(self._names[i], _ptr(a) if a is not None else None, b)
        self._arr = arr
        if fill is not None:
            self._fill = FILL_FN(lambda dst, nb, idx, ctx: fill(dst, nb, idx))
        else:
            self._fill = FILL_FN()
        h = VP()
        _check(lib().tidal_model_create(C.byref(self._cfg), arr, len(tensors), checkpoint.encode(),
                                        self._fill, None, world, rank, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().tidal_model_destroy(self.h)
            self.h = None


class Trace:
    def __init__(self, model: Model, tokens: Optional[np.ndarray] = None, device: int = -1):
        self.logits = None
        self.token = None
        self.cold_ms = None
        h = VP()
        if device < 0:
            _check(lib().tidal_trace(model.h, None, 0, -1, None, None, None, C.byref(h)))
        else:
            tok = np.ascontiguousarray(tokens, dtype=np.int32)
            self.logits = np.empty(model.vocab, np.float32)
            t = C.c_int32(0)
            ms = C.c_double(0)
            _check(lib().tidal_trace(model.h, tok.ctypes.data, len(tok), device,
                                     self.logits.ctypes.data, C.addressof(t), C.addressof(ms),
                                     C.byref(h)))
            self.token, self.cold_ms = t.value, ms.value
        self.h = h

    def dump(self) -> str:
        return _dump(lib().tidal_trace_dump, self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().tidal_trace_destroy(self.h)
            self.h = None


def template_opts(resident_bytes: int = U64_MAX, eq1: bool = False, t_ttft_s: float = 0.0,
                  b_pcie_Bps: float = 0.0, group_policy: int = GROUPS_PER_LAYER,
                  max_transfers: int = 300, max_tokens: int = 2048, device: int = -1,
                  comm=None) -> TemplateOpts:
    return TemplateOpts(resident_bytes, int(eq1), t_ttft_s, b_pcie_Bps, group_policy,
                        max_transfers, max_tokens, device, comm.h if comm is not None else None)


class Template:
    def __init__(self, model: Model, trace: Trace, opts: TemplateOpts,
                 shared: Optional[Tuple[List[int], int, int]] = None):
        """shared = (fds, shared_bytes, fingerprint) from another process's
        export(): map those template chunks read-only instead of building the
        prefix (refused with ERR_STRUCTURE if the fingerprint differs)."""
        h = VP()
        self._opts = opts
        if shared is None:
            _check(lib().tidal_template_create(model.h, trace.h, C.byref(opts), C.byref(h)))
        else:
            fds, nbytes, fp = shared
            arr = (C.c_int * len(fds))(*fds)
            _check(lib().tidal_template_import(model.h, trace.h, C.byref(opts), arr, len(fds),
                                               nbytes, fp, C.byref(h)))
        self.h = h
        self.vocab = model.vocab

    def export(self) -> Tuple[List[int], int, int]:
        """(fds of the chunks inside the resident prefix, shared_bytes,
        fingerprint); the caller owns the fds (pass them with socket.send_fds,
        then close)."""
        n = C.c_int(0)
        nb = C.c_uint64(0)
        fp = C.c_uint64(0)
        _check(lib().tidal_template_export(self.h, None, 0, C.byref(n), C.byref(nb), C.byref(fp)))
        arr = (C.c_int * max(1, n.value))()
        _check(lib().tidal_template_export(self.h, arr, n.value, C.byref(n), C.byref(nb),
                                           C.byref(fp)))
        return list(arr[:n.value]), nb.value, fp.value

    def resize(self, opts: TemplateOpts) -> None:
        _check(lib().tidal_template_resize(self.h, C.byref(opts)))

    def keep_alive(self) -> None:
        _check(lib().tidal_template_keep_alive(self.h))

    def set_load_order(self, order: int) -> None:
        _check(lib().tidal_set_load_order(self.h, order))

    def plan_dump(self, adapter: Optional["Adapter"] = None) -> str:
        return _dump(lib().tidal_plan_dump, self.h, adapter.h if adapter else None)

    def adapter_layout(self, rank: int, mask: int = 0x7F) -> Tuple[List[dict], int]:
        n = C.c_int(0)
        tot = C.c_uint64(0)
        _check(lib().tidal_adapter_layout(self.h, rank, mask, None, 0, C.byref(n), C.byref(tot)))
        slots = (Slot * max(1, n.value))()
        _check(lib().tidal_adapter_layout(self.h, rank, mask, slots, n.value, C.byref(n),
                                          C.byref(tot)))
        return ([{"name": s.name.decode(), "offset": s.offset, "bytes": s.bytes,
                  "rows": s.rows, "cols": s.cols} for s in slots[:n.value]], tot.value)

    def invoke(self, tokens: np.ndarray, adapter: Optional["Adapter"] = None,
               want_logits: bool = True) -> Tuple[int, Optional[np.ndarray], dict]:
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        logits = np.empty(self.vocab, np.float32) if want_logits else None
        t = C.c_int32(0)
        st = Stats()
        _check(lib().tidal_invoke_prefill(self.h, adapter.h if adapter else None, tok.ctypes.data,
                                          len(tok), logits.ctypes.data if want_logits else None,
                                          C.addressof(t), C.byref(st)))
        return t.value, logits, st.as_dict()

    def invoke_batch(self, tokens: np.ndarray, adapter: Optional["Adapter"] = None,
                     want_logits: bool = True) -> Tuple[np.ndarray, Optional[np.ndarray], dict]:
        """tokens [n_seqs, seq_len] -> (first tokens [n_seqs], logits [n_seqs, vocab], stats)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        if tok.ndim != 2:
            raise ValueError("tokens must be [n_seqs, seq_len]")
        B, S = tok.shape
        logits = np.empty((B, self.vocab), np.float32) if want_logits else None
        out = np.empty(B, np.int32)
        st = Stats()
        _check(lib().tidal_invoke_prefill_batch(self.h, adapter.h if adapter else None,
                                                tok.ctypes.data, B, S,
                                                logits.ctypes.data if want_logits else None,
                                                out.ctypes.data, C.byref(st)))
        return out, logits, st.as_dict()

    def enable_decode(self, max_new_tokens: int) -> None:
        """Allocate the KV cache; later single-prompt invocations fill it."""
        _check(lib().tidal_template_enable_decode(self.h, max_new_tokens))

    def decode(self, n_steps: int, adapter: Optional["Adapter"] = None,
               want_logits: bool = True) -> Tuple[np.ndarray, Optional[np.ndarray], dict]:
        """Greedy decode continuing the last single-prompt invoke():
        (tokens [n_steps], logits [n_steps, vocab] or None, stats)."""
        toks = np.empty(n_steps, np.int32)
        logits = np.empty((n_steps, self.vocab), np.float32) if want_logits else None
        st = DecodeStats()
        _check(lib().tidal_invoke_decode(self.h, adapter.h if adapter else None, n_steps,
                                         toks.ctypes.data,
                                         logits.ctypes.data if want_logits else None,
                                         C.byref(st)))
        return toks, logits, st.as_dict()

    def set_debug(self, flags: int, arg: int = -1) -> None:
        _check(lib().tidal_set_debug(self.h, flags, arg))

    def timeline(self) -> dict:
        """Copy-group end and op start times (ms) of the last DEBUG_TIMELINE invoke."""
        ng, no, end = C.c_int(0), C.c_int(0), C.c_double(0)
        _check(lib().tidal_timeline_read(self.h, None, 0, None, 0, C.byref(ng), C.byref(no),
                                         C.byref(end)))
        g = np.zeros(max(1, ng.value), np.float64)
        o = np.zeros(max(1, no.value), np.float64)
        _check(lib().tidal_timeline_read(self.h, g.ctypes.data, ng.value, o.ctypes.data, no.value,
                                         C.byref(ng), C.byref(no), C.byref(end)))
        return {"group_end_ms": g[:ng.value], "op_start_ms": o[:no.value], "end_ms": end.value}

    def set_allreduce_dtype(self, dtype: int) -> None:
        """DTYPE_F32 (default) or DTYPE_BF16 for the row-parallel allreduces."""
        _check(lib().tidal_set_allreduce_dtype(self.h, dtype))

    def profile(self, reset: bool = True) -> dict:
        n = C.c_int(0)
        arr = (KernelTime * 32)()
        _check(lib().tidal_profile_read(self.h, arr, 32, C.byref(n), int(reset)))
        return {k.name.decode(): {"ms": k.total_ms, "launches": k.launches, "flops": k.flops,
                                  "bytes": k.bytes} for k in arr[:n.value]}

    def checksum(self) -> int:
        v = C.c_uint64(0)
        _check(lib().tidal_template_checksum(self.h, C.byref(v)))
        return v.value

    def weight_ptr(self, name: str) -> int:
        p = VP()
        _check(lib().tidal_weight_ptr(self.h, name.encode(), C.byref(p)))
        return p.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().tidal_template_destroy(self.h)
            self.h = None


_allocator_refs = None


def set_device_allocator(alloc: Optional[Callable[[int, int], int]] = None,
                         free: Optional[Callable[[int, int], None]] = None) -> None:
    """Route the library's device allocations through alloc(bytes, device) ->
    ptr / free(ptr, device); no arguments: back to cudaMalloc."""
    global _allocator_refs
    if alloc is None:
        _check(lib().tidal_set_device_allocator(ALLOC_FN(), FREE_FN(), None))
        _allocator_refs = None
        return
    a = ALLOC_FN(lambda nb, dev, ctx: alloc(nb, dev) or None)
    f = FREE_FN(lambda p, dev, ctx: free(p, dev))
    _check(lib().tidal_set_device_allocator(a, f, None))
    _allocator_refs = (a, f)   # the C side keeps the function pointers


def use_torch_allocator() -> None:
    """Device memory from PyTorch's caching allocator (torch.cuda.caching_allocator_*)."""
    import torch
    set_device_allocator(lambda nb, dev: torch.cuda.caching_allocator_alloc(nb, dev),
                         lambda p, dev: torch.cuda.caching_allocator_delete(p))


class PinnedBuffer:
    """Page-locked host memory from tidal_host_alloc, viewable as numpy."""

    def __init__(self, nbytes: int):
        p = VP()
        _check(lib().tidal_host_alloc(nbytes, C.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def view(self, dtype=np.uint8) -> np.ndarray:
        buf = (C.c_uint8 * self.nbytes).from_address(self.ptr)
        return np.frombuffer(buf, dtype=np.uint8).view(dtype)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib().tidal_host_free(self.ptr)
            self.ptr = None


class Adapter:
    def __init__(self, tpl: Template, rank: int, scale: float, mask: int, buf: PinnedBuffer,
                 nbytes: int, checkpoint: str = "adapter"):
        self._buf = buf
        self._ck = checkpoint.encode()
        d = LoraDesc(rank, scale, mask, buf.ptr if buf is not None else None, nbytes, self._ck)
        h = VP()
        _check(lib().tidal_attach_lora(tpl.h, C.byref(d), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().tidal_adapter_destroy(self.h)
            self.h = None


class Comm:
    """TP communicator: NCCL (one process per GPU, `unique_id` from rank 0) or,
    with `local=<group name>`, the in-process ranks of one process (one thread
    per rank; ranks may share a GPU)."""

    def __init__(self, world: int, rank: int, unique_id: bytes = b"", device: int = 0,
                 local: Optional[str] = None):
        h = VP()
        if local is not None:
            _check(lib().tidal_comm_create_local(world, rank, local.encode(), device, C.byref(h)))
        else:
            idb = C.create_string_buffer(unique_id, 128)
            _check(lib().tidal_comm_create(world, rank, idb, device, C.byref(h)))
        self.h = h

    def selftest(self, n: int = 4096) -> None:
        """Run every collective on exact small-integer buffers (all ranks at once)."""
        _check(lib().tidal_comm_selftest(self.h, n))

    @staticmethod
    def unique_id() -> bytes:
        b = C.create_string_buffer(128)
        _check(lib().tidal_comm_unique_id(b))
        return b.raw

    def __del__(self):
        if getattr(self, "h", None):
            lib().tidal_comm_destroy(self.h)
            self.h = None


# ---------------- kernel-level entry points (device pointers) ----------------
def k_rmsnorm(X, g, Y, S, d, eps):
    _check(lib().tidal_k_rmsnorm(_ptr(X), _ptr(g), _ptr(Y), S, d, eps))


def k_embed(tok, E, X, S, d, row0, rows):
    _check(lib().tidal_k_embed(_ptr(tok), _ptr(E), _ptr(X), S, d, row0, rows))


def k_lora_shrink(X, M, K, A, T, r, scale):
    _check(lib().tidal_k_lora_shrink(_ptr(X), M, K, _ptr(A), _ptr(T), r, scale))


def k_attention(qkv, O, S, H, KV, hd):
    _check(lib().tidal_k_attention(_ptr(qkv), _ptr(O), S, H, KV, hd))


def k_attention_tc(qkv, vt, vt_ld, O, S, H, KV):
    _check(lib().tidal_k_attention_tc(_ptr(qkv), _ptr(vt), vt_ld, _ptr(O), S, H, KV))


def k_head(xlast, g, W, V, d, eps, logits, key):
    _check(lib().tidal_k_head(_ptr(xlast), _ptr(g), _ptr(W), V, d, eps, _ptr(logits), _ptr(key)))


def k_gemm(epi, A, Ws, seg_n, out, ldo, M, K, Ts=None, Bs=None, r=0, rope=None, head_dim=128):
    n = len(Ws)
    W = (VP * n)(*[_ptr(w) for w in Ws])
    sn = (C.c_int * n)(*seg_n)
    T = (VP * n)(*[_ptr(t) for t in Ts]) if Ts else None
    B = (VP * n)(*[_ptr(b) for b in Bs]) if Bs else None
    _check(lib().tidal_k_gemm(epi, _ptr(A), W, sn, len(seg_n), _ptr(out), ldo, M, K, T, B, r,
                              _ptr(rope), head_dim))
