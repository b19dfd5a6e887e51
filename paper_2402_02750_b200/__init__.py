"""B200-native KIVI KV-cache hot path (2-bit quantize-append + fused
dequant-attention decode).

The product is the in-tree C-ABI library ``libkivi_b200.so`` (CUDA kernels
for sm_100a, declared in ``include/kivi_b200.h``) plus the C++ drop-in facade
``libkivi_facade.so`` (the reference's ``kivi::`` API, ``include/kivi/``).
This module is a thin ctypes binding over the C-ABI used by the tests and
``bench.py``; PyTorch only provides device memory and streams.

There is no CPU fallback: importing works without a GPU, but every compute
call goes through the CUDA library and raises if it is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

__all__ = [
    "KiviError", "ShapeError", "UsageError", "ConfigError", "CudaError", "OutOfMemory",
    "CapacityError", "CacheConfig", "KVCache", "lib", "LIB_PATH", "HEADER_SYMBOLS",
    "quantize_matrix", "dequantize_matrix", "pack_codes", "unpack_codes",
    "reference_attention", "reload_tuning", "LayerStack", "Projection",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkivi_b200.so")
FACADE_PATH = os.path.join(_HERE, "libkivi_facade.so")


class KiviError(RuntimeError):
    """Base error; subclasses mirror reference errors.hpp:10-35."""


class ShapeError(KiviError):
    pass


class UsageError(KiviError):
    pass


class ConfigError(KiviError):
    pass


class CudaError(KiviError):
    pass


class OutOfMemory(KiviError):
    pass


class CapacityError(KiviError):
    pass


class BudgetError(KiviError):
    """reference BudgetError (errors.hpp:33-35): a memory budget was exceeded."""


class FormatError(KiviError):
    """reference FormatError (errors.hpp:25-30): malformed dump file; carries the
    byte offset of the failing field."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (at byte offset {offset})")
        self.byte_offset = offset


_ERRORS = {1: ShapeError, 2: UsageError, 3: ConfigError, 4: CudaError, 5: OutOfMemory,
           6: CapacityError}


class _Config(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("group_size", ctypes.c_int64),
                ("residual_length", ctypes.c_int64), ("head_dim", ctypes.c_int64)]


class _Info(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "n_units", "capacity_tokens", "total_tokens", "key_grouped_tokens",
        "key_residual_rows", "key_residual_capacity", "value_grouped_tokens",
        "value_residual_rows", "value_residual_capacity")] + [
        ("key_memory_bytes", ctypes.c_uint64), ("value_memory_bytes", ctypes.c_uint64),
        ("device_bytes", ctypes.c_uint64)]


class _UnitState(ctypes.Structure):
    _fields_ = [("key_packed", ctypes.c_void_p), ("key_zero", ctypes.c_void_p),
                ("key_scale", ctypes.c_void_p), ("key_residual", ctypes.c_void_p),
                ("value_packed", ctypes.c_void_p), ("value_zero", ctypes.c_void_p),
                ("value_scale", ctypes.c_void_p), ("value_residual", ctypes.c_void_p)]


P = ctypes.c_void_p
I32, I64, U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
# Every entry point declared in include/kivi_b200.h: name -> (restype, argtypes).
HEADER_SYMBOLS = {
    "kivi_last_error": (ctypes.c_char_p, []),
    "kivi_abi_version": (ctypes.c_int, []),
    "kivi_config_validate": (ctypes.c_int, [P]),
    "kivi_cache_create": (ctypes.c_int, [P, ctypes.c_int, I64, I64, P]),
    "kivi_cache_destroy": (ctypes.c_int, [P]),
    "kivi_cache_reserve": (ctypes.c_int, [P, I64, P]),
    "kivi_cache_clone": (ctypes.c_int, [P, P, P]),
    "kivi_cache_get_info": (ctypes.c_int, [P, P]),
    "kivi_prefill": (ctypes.c_int, [P, P, P, I64, P]),
    "kivi_append": (ctypes.c_int, [P, P, P, P]),
    "kivi_attend": (ctypes.c_int, [P, P, I32, P, P, I32, P]),
    "kivi_decode": (ctypes.c_int, [P, P, P, P, I32, P, P, I32, P]),
    "kivi_prefill_host": (ctypes.c_int, [P, P, P, I64, P]),
    "kivi_append_host": (ctypes.c_int, [P, P, P, P]),
    "kivi_decode_host": (ctypes.c_int, [P, P, P, P, I32, P, P, I32, P]),
    "kivi_host_join": (ctypes.c_int, [P, P]),
    "kivi_decode_layers": (ctypes.c_int, [P, I32, P, P, P, I32, P, I32, P]),
    "kivi_decode_layers_host": (ctypes.c_int, [P, I32, P, P, P, I32, P, I32, P]),
    "kivi_step_graph_stats": (ctypes.c_int, [P, P, P]),
    "kivi_proj_create": (ctypes.c_int, [ctypes.c_int, I64, I64, P, P, P, P, P]),
    "kivi_proj_destroy": (ctypes.c_int, [P]),
    "kivi_proj_gemm": (ctypes.c_int, [P, P, I64, P, P, P, I64, P]),
    "kivi_proj_append": (ctypes.c_int, [P, P, P, I64, P, P]),
    "kivi_export_unit": (ctypes.c_int, [P, I64, P, P]),
    "kivi_import_unit": (ctypes.c_int, [P, I64, I64, I64, I64, P, P]),
    "kivi_materialize": (ctypes.c_int, [P, P, P, P]),
    "kivi_quantize_matrix": (ctypes.c_int, [P, I64, I64, I32, I64, ctypes.c_int, P, P, P, P]),
    "kivi_dequantize_matrix": (ctypes.c_int, [P, P, P, I64, I64, I32, I64, ctypes.c_int, P, P]),
    "kivi_quantize_codes": (ctypes.c_int, [P, I64, I64, I32, I64, ctypes.c_int, P, P, P, P]),
    "kivi_quantize_group": (ctypes.c_int, [P, I64, I32, P, P, P, P, P]),
    "kivi_dequantize_codes": (ctypes.c_int, [P, P, P, I64, I64, I64, ctypes.c_int, P, P]),
    "kivi_pack_codes": (ctypes.c_int, [P, I64, I32, P, P]),
    "kivi_unpack_codes": (ctypes.c_int, [P, I64, I32, P, P]),
    "kivi_reference_attention": (ctypes.c_int, [P, I64, P, P, I64, I64, I32, P, P]),
    "kivi_reload_tuning": (ctypes.c_int, []),
    "kivi_set_attend_path": (ctypes.c_int, [P, I32]),
    "kivi_profile_enable": (ctypes.c_int, [P, I32]),
    "kivi_profile_read": (ctypes.c_int, [P, P, P, P]),
    "kivi_attend_bytes": (ctypes.c_int, [P, I32, P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Loads the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2402_02750_b200` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in HEADER_SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        msg = lib().kivi_last_error().decode(errors="replace")
        raise _ERRORS.get(status, KiviError)(msg)


def _torch():
    import torch
    return torch


def reload_tuning() -> None:
    """Re-reads the KIVI_* routing knobs from the environment (kivi_reload_tuning)."""
    _check(lib().kivi_reload_tuning())


def _stream_ptr(stream=None, device=None) -> int:
    """The given stream, else torch's current stream OF `device` (the cache's
    device, which need not be the current one)."""
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _dptr(t, device=None) -> int:
    if t is None:
        return None
    if not t.is_cuda:
        raise UsageError("expected a CUDA tensor")
    if device is not None and t.device.index != device:
        raise UsageError(f"tensor on cuda:{t.device.index}, cache on cuda:{device}")
    if not t.is_contiguous():
        raise UsageError("expected a contiguous tensor")
    return t.data_ptr()


@dataclass(frozen=True)
class CacheConfig:
    """Mirrors reference CacheConfig (kv_cache.hpp:9-18)."""
    bits: int = 2
    group_size: int = 32
    residual_length: int = 128
    head_dim: int = 128

    def _c(self) -> _Config:
        return _Config(self.bits, self.group_size, self.residual_length, self.head_dim)

    def validate(self) -> None:
        c = self._c()
        _check(lib().kivi_config_validate(ctypes.byref(c)))


class KVCache:
    """n_units lockstep KIVI caches (one per (batch, kv-head) of a layer).

    Device-tensor methods enqueue on the current torch stream and return
    without synchronising; ``*_host`` methods take numpy arrays.
    """

    def __init__(self, cfg: CacheConfig, n_units: int, capacity_tokens: int = 0,
                 device: int | None = None):
        torch = _torch()
        self.cfg = cfg
        self.n_units = int(n_units)
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = ctypes.c_void_p()
        c = cfg._c()
        _check(lib().kivi_cache_create(ctypes.byref(c), self.device, self.n_units,
                                       int(capacity_tokens), ctypes.byref(h)))
        self._h = h

    @property
    def _decode_fn(self):
        return lib().kivi_decode

    @classmethod
    def _wrap(cls, cfg, n_units, device, handle):
        obj = cls.__new__(cls)
        obj.cfg, obj.n_units, obj.device, obj._h = cfg, n_units, device, handle
        return obj

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().kivi_cache_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state ----------------------------------------------------------
    def info(self) -> dict:
        i = _Info()
        _check(lib().kivi_cache_get_info(self._h, ctypes.byref(i)))
        return {n: getattr(i, n) for n, _ in _Info._fields_}

    @property
    def total_tokens(self) -> int:
        return self.info()["total_tokens"]

    def reserve(self, capacity_tokens: int) -> None:
        _check(lib().kivi_cache_reserve(self._h, int(capacity_tokens), _stream_ptr(None, self.device)))

    def clone(self) -> "KVCache":
        h = ctypes.c_void_p()
        _check(lib().kivi_cache_clone(self._h, _stream_ptr(None, self.device), ctypes.byref(h)))
        return KVCache._wrap(self.cfg, self.n_units, self.device, h)

    def set_attend_path(self, path: str) -> None:
        _check(lib().kivi_set_attend_path(self._h, {"auto": 0, "generic": 1, "fast": 2}[path]))

    # ---- hot path (device tensors) ---------------------------------------
    def prefill(self, keys, values) -> None:
        """keys/values: [n_units, l, d] fp32 CUDA tensors."""
        self._shape(keys, 3, "prefill keys")
        self._shape(values, 3, "prefill values")
        if keys.shape != values.shape:
            raise ShapeError("prefill: key/value token counts differ")
        _check(lib().kivi_prefill(self._h, _dptr(keys, self.device), _dptr(values, self.device), int(keys.shape[1]),
                                  _stream_ptr(None, self.device)))

    def append(self, t_k, t_v) -> None:
        """t_k, t_v: [n_units, d] fp32 CUDA tensors."""
        self._rows(t_k, "append_token key")
        self._rows(t_v, "append_token value")
        _check(lib().kivi_append(self._h, _dptr(t_k, self.device), _dptr(t_v, self.device), _stream_ptr(None, self.device)))

    def attend(self, q, q_per_kv: int = 1, weights: bool = False, scale_logits: bool = True,
               out=None):
        torch = _torch()
        d = self.cfg.head_dim
        if q.numel() != self.n_units * q_per_kv * d or q.dtype != torch.float32:
            raise ShapeError(f"query must be [n_units, q_per_kv, {d}] fp32")
        if out is None:
            out = torch.empty((self.n_units, q_per_kv, d), device=q.device, dtype=torch.float32)
        w = None
        if weights:
            w = torch.empty((self.n_units, q_per_kv, self.total_tokens), device=q.device,
                            dtype=torch.float32)
        _check(lib().kivi_attend(self._h, _dptr(q.contiguous(), self.device), int(q_per_kv), _dptr(out, self.device),
                                 _dptr(w, self.device), int(bool(scale_logits)), _stream_ptr(None, self.device)))
        return (out, w) if weights else out

    def decode(self, q, t_k, t_v, q_per_kv: int = 1, weights: bool = False,
               scale_logits: bool = True, out=None):
        """Reference decode_attention: append, then attend (attention.cpp:26-100).
        One C-ABI call (kivi_decode); the serving loop calls this per layer, so
        the host path is kept to a few checks."""
        if weights:
            self.append(t_k, t_v)
            return self.attend(q, q_per_kv=q_per_kv, weights=True, scale_logits=scale_logits,
                               out=out)
        torch = _torch()
        d, U = self.cfg.head_dim, self.n_units
        if t_k.numel() != U * d or t_v.numel() != U * d or t_k.dtype != torch.float32 \
                or t_v.dtype != torch.float32:
            raise ShapeError(f"append_token: expected 1x{d} rows per unit")
        if q.numel() != U * q_per_kv * d or q.dtype != torch.float32:
            raise ShapeError(f"query must be [n_units, q_per_kv, {d}] fp32")
        if out is None:
            out = torch.empty((U, q_per_kv, d), device=q.device, dtype=torch.float32)
        _check(self._decode_fn(self._h, _dptr(q, self.device), _dptr(t_k, self.device), _dptr(t_v, self.device), int(q_per_kv),
                               _dptr(out, self.device), None, int(bool(scale_logits)),
                               torch.cuda.current_stream(self.device).cuda_stream))
        return out

    # ---- host-buffer path -------------------------------------------------
    def prefill_host(self, keys, values) -> None:
        import numpy as np
        k = np.ascontiguousarray(keys, dtype=np.float32)
        v = np.ascontiguousarray(values, dtype=np.float32)
        if k.shape != v.shape or k.ndim != 3:
            raise ShapeError("prefill: keys/values must both be [n_units, l, d]")
        _check(lib().kivi_prefill_host(self._h, k.ctypes.data, v.ctypes.data, k.shape[1],
                                       _stream_ptr(None, self.device)))

    def decode_host(self, q, t_k, t_v, out, q_per_kv: int = 1, weights=None,
                    scale_logits: bool = True, stream=None) -> None:
        """All arguments are host buffers (numpy, ideally pinned); the copies are
        enqueued with the kernels on `stream`, the result copy on the cache's own
        copy stream: call host_join(stream) and synchronise before reading."""
        _check(lib().kivi_decode_host(
            self._h, _hptr(q), _hptr(t_k), _hptr(t_v), int(q_per_kv), _hptr(out),
            _hptr(weights) if weights is not None else None, int(bool(scale_logits)),
            _stream_ptr(stream, self.device)))

    def host_join(self, stream=None) -> None:
        """Orders `stream` after every result copy decode_host has enqueued."""
        _check(lib().kivi_host_join(self._h, _stream_ptr(stream, self.device)))

    # ---- parity helpers -----------------------------------------------------
    def export_unit(self, unit: int) -> dict:
        import numpy as np
        i = self.info()
        d, G, B = self.cfg.head_dim, self.cfg.group_size, self.cfg.bits
        kg, vg = i["key_grouped_tokens"], i["value_grouped_tokens"]
        bufs = {
            "key_packed": np.zeros(((kg * d * B + 7) // 8,), np.uint8),
            "key_zero": np.zeros((kg * d // G,), np.float64),
            "key_scale": np.zeros((kg * d // G,), np.float64),
            "key_residual": np.zeros((i["key_residual_rows"], d), np.float32),
            "value_packed": np.zeros(((vg * d * B + 7) // 8,), np.uint8),
            "value_zero": np.zeros((vg * d // G,), np.float64),
            "value_scale": np.zeros((vg * d // G,), np.float64),
            "value_residual": np.zeros((i["value_residual_rows"], d), np.float32),
        }
        st = _UnitState(*[b.ctypes.data if b.size else None for b in bufs.values()])
        _check(lib().kivi_export_unit(self._h, int(unit), ctypes.byref(st), _stream_ptr(None, self.device)))
        return bufs

    def import_unit(self, unit: int, total_tokens: int, key_residual_capacity: int,
                    value_residual_capacity: int, state: dict) -> None:
        import numpy as np
        order = ["key_packed", "key_zero", "key_scale", "key_residual", "value_packed",
                 "value_zero", "value_scale", "value_residual"]
        dt = [np.uint8, np.float64, np.float64, np.float32] * 2
        arrs = [np.ascontiguousarray(state[k], dtype=t) for k, t in zip(order, dt)]
        st = _UnitState(*[a.ctypes.data if a.size else None for a in arrs])
        _check(lib().kivi_import_unit(self._h, int(unit), int(total_tokens),
                                      int(key_residual_capacity), int(value_residual_capacity),
                                      ctypes.byref(st), _stream_ptr(None, self.device)))

    def materialize(self):
        torch = _torch()
        l, d = self.total_tokens, self.cfg.head_dim
        k = torch.empty((self.n_units, l, d), device=f"cuda:{self.device}", dtype=torch.float32)
        v = torch.empty_like(k)
        _check(lib().kivi_materialize(self._h, _dptr(k, self.device), _dptr(v, self.device), _stream_ptr(None, self.device)))
        return k, v

    # ---- measurement hooks ---------------------------------------------------
    def profile_enable(self, on=True) -> None:
        """on: False/0 = off; True/1 = time every attend launch; k > 1 = time
        every k-th launch (include/kivi_b200.h kivi_profile_enable)."""
        k = int(on) if not isinstance(on, bool) else int(on)
        if k < 0:
            raise UsageError("profile stride must be >= 0")
        _check(lib().kivi_profile_enable(self._h, k))

    def profile_read(self):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        tot = ctypes.c_int64()
        _check(lib().kivi_profile_read(self._h, ctypes.byref(ms), ctypes.byref(n),
                                       ctypes.byref(tot)))
        return ms.value, n.value, tot.value

    def attend_bytes_per_unit(self, q_per_kv: int = 1) -> int:
        b = ctypes.c_uint64()
        _check(lib().kivi_attend_bytes(self._h, int(q_per_kv), ctypes.byref(b)))
        return b.value

    # ---- helpers ---------------------------------------------------------------
    def _shape(self, t, ndim, what):
        torch = _torch()
        if t.dim() != ndim or t.shape[0] != self.n_units or t.shape[-1] != self.cfg.head_dim \
                or t.dtype != torch.float32:
            raise ShapeError(f"{what}: expected [{self.n_units}, ..., {self.cfg.head_dim}] fp32")

    def _rows(self, t, what):
        torch = _torch()
        if t.numel() != self.n_units * self.cfg.head_dim or t.dtype != torch.float32:
            raise ShapeError(f"{what}: expected 1x{self.cfg.head_dim} rows per unit")


class LayerStack:
    """The caches of a model's layers (same units / head_dim / device), decoded
    one whole step per C-ABI call (kivi_decode_layers[_host]): the host loop
    over layers runs in native code."""

    def __init__(self, caches):
        self.caches = list(caches)
        if not self.caches:
            raise UsageError("LayerStack: no caches")
        self.device = self.caches[0].device
        self._arr = (ctypes.c_void_p * len(self.caches))(*[c._h.value for c in self.caches])

    def decode(self, q, t_k, t_v, out, q_per_kv: int = 1, scale_logits: bool = True) -> None:
        """Device tensors: q/out [L, U, q_per_kv, d], t_k/t_v [L, U, d]."""
        dv = self.device
        _check(lib().kivi_decode_layers(self._arr, len(self.caches), _dptr(q, dv), _dptr(t_k, dv),
                                        _dptr(t_v, dv), int(q_per_kv), _dptr(out, dv),
                                        int(bool(scale_logits)), _stream_ptr(None, dv)))

    def decode_host(self, q, t_k, t_v, out, q_per_kv: int = 1, scale_logits: bool = True,
                    stream=None) -> None:
        """Host buffers (pinned for speed); returns with the outputs in `out`."""
        _check(lib().kivi_decode_layers_host(self._arr, len(self.caches), _hptr(q), _hptr(t_k),
                                             _hptr(t_v), int(q_per_kv), _hptr(out),
                                             int(bool(scale_logits)),
                                             _stream_ptr(stream, self.device)))

    def bind_host_step(self, q, t_k, t_v, out, q_per_kv: int = 1, scale_logits: bool = True,
                       stream=None):
        """decode_host over fixed (pinned) host buffers, arguments resolved once:
        returns a no-argument callable for a serving loop that refills the same
        buffers every step (a latency-bound step then pays only the C call)."""
        f = lib().kivi_decode_layers_host
        args = (self._arr, len(self.caches), _hptr(q), _hptr(t_k), _hptr(t_v), int(q_per_kv),
                _hptr(out), int(bool(scale_logits)), _stream_ptr(stream, self.device))

        def step():
            st = f(*args)
            if st:
                _check(st)
        return step


class Projection:
    """One layer's q/k/v projection (reference workload.cpp:230-232, x @ W) on
    the tcgen05 tensor cores in 3xTF32, optionally fused with the KV-cache
    append (kivi_proj_append).  w_q, w_k, w_v: [hidden_in, hidden_out] fp32
    CUDA tensors (copied and transposed once)."""

    def __init__(self, w_q, w_k, w_v):
        self.hidden_in, self.hidden_out = int(w_q.shape[0]), int(w_q.shape[1])
        self.device = w_q.device.index
        h = ctypes.c_void_p()
        _check(lib().kivi_proj_create(self.device, self.hidden_in, self.hidden_out,
                                      _dptr(w_q.contiguous(), self.device),
                                      _dptr(w_k.contiguous(), self.device),
                                      _dptr(w_v.contiguous(), self.device),
                                      _stream_ptr(None, self.device), ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().kivi_proj_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def gemm(self, x, seq: int = 0):
        """x: [n, hidden_in] -> (q, k, v) [n, hidden_out]; seq > 0: per-unit
        [n // seq * heads, seq, 128] (the layout KVCache.prefill takes)."""
        torch = _torch()
        n = int(x.shape[0])
        shape = (n, self.hidden_out) if seq == 0 else \
            (n // seq * (self.hidden_out // 128), seq, 128)
        outs = [torch.empty(shape, device=x.device, dtype=torch.float32) for _ in range(3)]
        dv = self.device
        _check(lib().kivi_proj_gemm(self._h, _dptr(x.contiguous(), dv), n,
                                    *[_dptr(o, dv) for o in outs], int(seq),
                                    _stream_ptr(None, dv)))
        return tuple(outs)

    def append(self, cache, x, q_out=None):
        """Projection of the decode token rows x [n, hidden_in] fused with the
        append into `cache` (n * heads units); returns q [n * heads, 1, 128]."""
        torch = _torch()
        n = int(x.shape[0])
        if q_out is None:
            q_out = torch.empty((n * (self.hidden_out // 128), 1, 128), device=x.device,
                                dtype=torch.float32)
        dv = self.device
        _check(lib().kivi_proj_append(self._h, cache._h, _dptr(x.contiguous(), dv), n,
                                      _dptr(q_out, dv), _stream_ptr(None, dv)))
        return q_out


def step_graph_stats(device=None) -> dict:
    """kivi_step_graph_stats of this thread on `device` (default: current)."""
    torch = _torch()
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        _check(lib().kivi_step_graph_stats(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"replayed": a.value, "reinstantiated": b.value, "capture_failed": c.value}


def _hptr(a):
    import numpy as np
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise UsageError("host buffer must be C-contiguous")
        return a.ctypes.data
    # torch CPU tensor (possibly pinned)
    return a.data_ptr()


# ---- standalone quantizer (reference quantize.hpp:35-96) ---------------------

def quantize_matrix(m, bits: int, group_size: int, per_channel: bool):
    """QuantizedTensor::quantize on the GPU: returns (packed u8, zero f64, scale f64)
    as CUDA tensors."""
    torch = _torch()
    rows, cols = m.shape
    nbytes = (rows * cols * bits + 7) // 8
    ng = rows * cols // group_size if group_size > 0 else 0
    packed = torch.zeros((nbytes,), dtype=torch.uint8, device=m.device)
    z = torch.zeros((max(ng, 1),), dtype=torch.float64, device=m.device)
    s = torch.zeros((max(ng, 1),), dtype=torch.float64, device=m.device)
    _check(lib().kivi_quantize_matrix(_dptr(m.contiguous()), rows, cols, bits, group_size,
                                      1 if per_channel else 0, _dptr(packed), _dptr(z),
                                      _dptr(s), _stream_ptr(None, m.device)))
    return packed, z[:ng], s[:ng]


def dequantize_matrix(packed, zero, scale, rows, cols, bits, group_size, per_channel):
    torch = _torch()
    out = torch.empty((rows, cols), dtype=torch.float32, device=packed.device)
    _check(lib().kivi_dequantize_matrix(_dptr(packed), _dptr(zero), _dptr(scale), rows, cols,
                                        bits, group_size, 1 if per_channel else 0, _dptr(out),
                                        _stream_ptr(None, packed.device)))
    return out


def pack_codes(codes, bits: int):
    torch = _torch()
    n = codes.numel()
    out = torch.zeros(((n * bits + 7) // 8,), dtype=torch.uint8, device=codes.device)
    _check(lib().kivi_pack_codes(_dptr(codes), n, bits, _dptr(out), _stream_ptr(None, codes.device)))
    return out


def unpack_codes(packed, n: int, bits: int):
    torch = _torch()
    out = torch.zeros((n,), dtype=torch.uint8, device=packed.device)
    _check(lib().kivi_unpack_codes(_dptr(packed), n, bits, _dptr(out), _stream_ptr(None, packed.device)))
    return out


def reference_attention(q, K, V, scale_logits: bool = True):
    """Reference reference_attention (attention.cpp:16-24) on the GPU."""
    torch = _torch()
    nq, d = q.shape
    l = K.shape[0]
    out = torch.empty((nq, d), dtype=torch.float32, device=q.device)
    _check(lib().kivi_reference_attention(_dptr(q.contiguous()), nq, _dptr(K.contiguous()),
                                          _dptr(V.contiguous()), l, d, int(bool(scale_logits)),
                                          _dptr(out), _stream_ptr(None, q.device)))
    return out
