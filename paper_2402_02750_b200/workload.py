"""The reference's workload layer on the GPU.

Mirrors reference proj/include/kivi/workload.hpp / src/workload.cpp:
  * WorkloadSpec, preset_spec, preset_names        (workload.hpp:14-36, workload.cpp:12-36)
  * fp_cache_bytes, estimate_memory               (workload.cpp:38-86): closed-form accounting
  * max_batch_at_budget                           (workload.cpp:88-114)
  * run_decode_benchmark                          (workload.cpp:145-271): prefill + gen_len
    decode steps over synthetic projections, one cache per (batch, layer, head)

run_decode_benchmark is the reference's only in-tree caller of the hot path.  Here it
drives the B200 library the way a serving loop would.  Per layer and step, ONE launch
(kivi_proj_append, tcgen05 3xTF32 tensor cores) projects every sequence's token
(t @ W_q/k/v, workload.cpp:230-232) and appends the new key/value rows straight into the
caches (unit = batch * kv_heads + head) -- the value FIFO pop is quantized in the GEMM
epilogue -- then one kivi_attend per layer reads the q rows it wrote.  The prompt's
projections use the same kernel (kivi_proj_gemm, per-unit output layout) before the bulk
prefill.  Shapes the fused kernel does not cover (head_dim != 128, hidden % 32 != 0,
group size != 32, bits not in {2, 4}) use cuBLAS fp32 GEMMs and kivi_decode.
Peak cache bytes are counted from the live device states (kivi_cache_get_info, the
reference's memory_bytes) and checked against the budget after prefill and every step,
as the reference does (workload.cpp:175-192).

Differences, by design: the reference decodes one (batch element, layer, head) state at
a time and times each batch element's step; here a step decodes the whole batch at once
and its latency (CUDA events) is the step's.  BenchMode "fp" (the 16-bit baseline) runs
the same loop with exact attention over fp32 device caches.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

from . import BudgetError, CacheConfig, ConfigError, KVCache, Projection, UsageError


@dataclass(frozen=True)
class WorkloadSpec:
    """reference WorkloadSpec (workload.hpp:14-24)."""
    batch: int = 1
    prompt_len: int = 161   # ShareGPT mean prompt length
    gen_len: int = 338      # ShareGPT mean output length
    layers: int = 2
    kv_heads: int = 2
    head_dim: int = 64

    def hidden(self) -> int:
        return self.kv_heads * self.head_dim

    def total_len(self) -> int:
        return self.prompt_len + self.gen_len

    def validate(self) -> None:  # workload.cpp:12-17
        if min(self.batch, self.prompt_len, self.layers, self.kv_heads, self.head_dim) < 1:
            raise ConfigError("workload counts must be >= 1")
        if self.gen_len < 0:
            raise ConfigError("gen_len must be >= 0")


_PRESETS = {  # workload.cpp:19-36
    "opt175b": WorkloadSpec(batch=512, prompt_len=512, gen_len=32, layers=96, kv_heads=96,
                            head_dim=128),
    "llama2-7b": WorkloadSpec(batch=16, prompt_len=3968, gen_len=128, layers=32, kv_heads=32,
                              head_dim=128),
    "sharegpt-tiny": WorkloadSpec(),
}


def preset_names():
    return list(_PRESETS)


def preset_spec(name: str) -> WorkloadSpec:
    if name not in _PRESETS:
        raise UsageError(f'unknown preset "{name}"')
    return _PRESETS[name]


@dataclass(frozen=True)
class MemoryEstimate:
    """reference MemoryEstimate (workload.hpp:29-36)."""
    fp_bytes: int
    kivi_bytes: int
    code_bytes: int
    scale_zero_bytes: int
    residual_bytes: int
    compression_ratio: float


def fp_cache_bytes(spec: WorkloadSpec) -> int:
    """2 caches x b x l x hidden x layers x 2 bytes (workload.cpp:38-45)."""
    spec.validate()
    return 2 * spec.batch * spec.total_len() * spec.hidden() * spec.layers * 2


def _check_cfg(spec: WorkloadSpec, cfg: CacheConfig, what: str) -> None:
    cfg.validate()
    if cfg.head_dim != spec.head_dim:
        raise ConfigError(f"{what}: cfg.head_dim must match spec.head_dim")


def estimate_memory(spec: WorkloadSpec, cfg: CacheConfig) -> MemoryEstimate:
    """Closed-form peak cache bytes of a full prefill + decode run (workload.cpp:47-86)."""
    spec.validate()
    _check_cfg(spec, cfg, "estimate_memory")
    l, lp, d = spec.total_len(), spec.prompt_len, spec.head_dim
    G, R, B = cfg.group_size, cfg.residual_length, cfg.bits
    key_grouped = l - l % R
    key_flushed = (l // R) > (lp // R)
    key_res_rows = R if key_flushed else l % R
    value_res_rows = min(l, R)
    value_grouped = l - value_res_rows
    n = spec.batch * spec.layers * spec.kv_heads
    code = ((key_grouped * d * B + 7) // 8 + (value_grouped * d * B + 7) // 8) * n
    sz = 4 * (key_grouped * d // G + value_grouped * d // G) * n
    res = 2 * (key_res_rows + value_res_rows) * d * n
    kivi = code + sz + res
    fp = fp_cache_bytes(spec)
    return MemoryEstimate(fp, kivi, code, sz, res, fp / kivi if kivi else 0.0)


def max_batch_at_budget(spec: WorkloadSpec, budget_bytes: int, mode: str,
                        cfg: CacheConfig) -> int:
    """Largest batch whose estimated peak fits the budget (workload.cpp:88-114)."""
    def bytes_at(b):
        s = replace(spec, batch=b)
        return fp_cache_bytes(s) if mode == "fp" else estimate_memory(s, cfg).kivi_bytes
    per_request = bytes_at(1)
    if per_request > budget_bytes:
        raise BudgetError(f"budget {budget_bytes} bytes below single-request footprint of "
                          f"{per_request} bytes")
    lo, hi = 1, budget_bytes // per_request + 1
    while lo < hi:
        mid = lo + (hi - lo + 1) // 2
        if bytes_at(mid) <= budget_bytes:
            lo = mid
        else:
            hi = mid - 1
    return lo


@dataclass
class BenchReport:
    """reference BenchReport (workload.hpp:57-67)."""
    mode: str = "kivi"
    decode_steps: int = 0
    tokens_per_sec: float = 0.0
    p50_ms: float = 0.0
    p90_ms: float = 0.0
    p99_ms: float = 0.0
    peak_cache_bytes: int = 0
    output_checksum: float = 0.0
    output_abs_sum: float = 0.0   # not in the reference: scale for checksum tolerances


def _percentile(sorted_ms, q):  # workload.cpp:135-141
    if not sorted_ms:
        return 0.0
    idx = int(math.ceil(q * len(sorted_ms))) - 1
    return sorted_ms[min(max(idx, 0), len(sorted_ms) - 1)]


def run_decode_benchmark(spec: WorkloadSpec, cfg: CacheConfig, seed: int = 0,
                         mode: str = "kivi", budget_bytes: int | None = None, data=None,
                         device: int | None = None,
                         fused_projection: bool | None = None) -> BenchReport:
    """Reference run_decode_benchmark (workload.cpp:145-271) on the GPU.

    data: optional (weights [layers, 3, hidden, hidden], prompts [batch, prompt_len, hidden],
    tokens [gen_len, batch, hidden]) fp32 arrays, e.g. the reference's own draws; by
    default they are drawn on the device from `seed` (N(0, 1), weights scaled by
    1/sqrt(hidden) as SyntheticLayer does, workload.cpp:116-122).
    fused_projection: None = the tensor-core projection fused with the append
    wherever its shape constraints hold; False = cuBLAS GEMMs + kivi_decode.
    """
    import torch
    spec.validate()
    _check_cfg(spec, cfg, "run_decode_benchmark")
    if mode not in ("kivi", "fp"):
        raise UsageError(f"unknown mode {mode!r}")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    H, d, hid, Bt = spec.kv_heads, spec.head_dim, spec.hidden(), spec.batch
    U = Bt * H
    if data is None:
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        W = torch.randn((spec.layers, 3, hid, hid), generator=g, device=dev) / math.sqrt(hid)
        P = torch.randn((Bt, spec.prompt_len, hid), generator=g, device=dev)
        T = torch.randn((spec.gen_len, Bt, hid), generator=g, device=dev)
    else:
        W, P, T = (torch.as_tensor(a, dtype=torch.float32).to(dev) for a in data)

    def units(x):  # [batch, n, hidden] -> [batch * heads, n, d]
        n = x.shape[1]
        return x.view(Bt, n, H, d).permute(0, 2, 1, 3).reshape(U, n, d).contiguous()

    # the fused tensor-core projection + append (kernels_project.cuh)
    fused = (mode == "kivi" and d == 128 and hid % 32 == 0 and cfg.group_size == 32
             and cfg.bits in (2, 4) and cfg.head_dim == 128 and fused_projection is not False)
    if fused_projection and not fused:
        raise ConfigError("fused projection needs head_dim 128, hidden % 32 == 0, group 32, "
                          "2 or 4 bits, mode 'kivi'")
    projs = [Projection(W[ly, 0], W[ly, 1], W[ly, 2]) for ly in range(spec.layers)] \
        if fused else []
    caches, fp = [], []
    for ly in range(spec.layers):
        if fused:
            _, K, V = projs[ly].gemm(P.reshape(Bt * spec.prompt_len, hid), seq=spec.prompt_len)
        else:
            K = units(torch.matmul(P, W[ly, 1]))
            V = units(torch.matmul(P, W[ly, 2]))
        if mode == "kivi":
            c = KVCache(cfg, U, capacity_tokens=spec.total_len(), device=dev.index)
            c.prefill(K, V)
            caches.append(c)
        else:
            fp.append([K, V])

    def counted_bytes():
        if mode == "kivi":
            tot = 0
            for c in caches:
                i = c.info()
                tot += (i["key_memory_bytes"] + i["value_memory_bytes"]) * U
            return tot
        return sum(2 * (k.numel() + v.numel()) for k, v in fp)

    def check_budget(step):
        if budget_bytes is None:
            return
        used = counted_bytes()
        if used > budget_bytes:
            raise BudgetError(f"memory budget exceeded at {step}: {used} > {budget_bytes} bytes")

    check_budget("prefill")
    stream = torch.cuda.current_stream(dev)
    checksum = torch.zeros((), dtype=torch.float64, device=dev)
    abs_sum = torch.zeros((), dtype=torch.float64, device=dev)
    events = []
    scale = 1.0 / math.sqrt(d)
    for step in range(spec.gen_len):
        t = T[step]                                   # [batch, hidden]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for ly in range(spec.layers):
            if fused:
                out = caches[ly].attend(projs[ly].append(caches[ly], t))
                checksum += out.double().sum()
                abs_sum += out.double().abs().sum()
                continue
            q, k, v = (torch.matmul(t, W[ly, i]).view(U, 1, d) for i in range(3))
            if mode == "kivi":
                out = caches[ly].decode(q, k.view(U, d), v.view(U, d))
            else:
                Kc = torch.cat([fp[ly][0], k], dim=1)
                Vc = torch.cat([fp[ly][1], v], dim=1)
                fp[ly] = [Kc, Vc]
                w = torch.softmax(torch.matmul(q, Kc.transpose(1, 2)) * scale, dim=-1)
                out = torch.matmul(w, Vc)
            checksum += out.double().sum()
            abs_sum += out.double().abs().sum()
        e1.record(stream)
        events.append((e0, e1))
        check_budget(f"decode step {step + 1}")
    torch.cuda.synchronize(dev)
    lat = sorted(a.elapsed_time(b) for a, b in events)
    total_s = sum(lat) / 1e3
    rep = BenchReport(mode=mode, decode_steps=spec.gen_len,
                      tokens_per_sec=(Bt * spec.gen_len / total_s) if total_s > 0 else 0.0,
                      p50_ms=_percentile(lat, 0.50), p90_ms=_percentile(lat, 0.90),
                      p99_ms=_percentile(lat, 0.99), peak_cache_bytes=counted_bytes(),
                      output_checksum=float(checksum.item()),
                      output_abs_sum=float(abs_sum.item()))
    for c in caches:
        c.close()
    for p_ in projs:
        p_.close()
    return rep


# ---- native driver (libkivi_driver.so, include/kivi_driver.h) -----------------

DRIVER_PATH = __import__("os").path.join(__import__("os").path.dirname(__file__),
                                         "libkivi_driver.so")
DRIVER_SYMBOLS = ("kivi_run_decode_benchmark", "kivi_driver_last_error")
_driver = None


def driver_lib():
    """libkivi_driver.so: the C++ decode driver over the C-ABI (raises if not built)."""
    import ctypes
    global _driver
    if _driver is None:
        from . import lib
        lib()  # libkivi_b200.so first (the driver links it)
        import os
        if not os.path.exists(DRIVER_PATH):
            raise ImportError(f"{DRIVER_PATH} is missing: build it with "
                              "`make -C paper_2402_02750_b200`")
        L = ctypes.CDLL(DRIVER_PATH)
        L.kivi_run_decode_benchmark.restype = ctypes.c_int
        L.kivi_run_decode_benchmark.argtypes = [
            ctypes.POINTER(_Spec), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
            ctypes.POINTER(_Report)]
        L.kivi_driver_last_error.restype = ctypes.c_char_p
        L.kivi_driver_last_error.argtypes = []
        _driver = L
    return _driver


import ctypes as _ct  # noqa: E402


class _Spec(_ct.Structure):
    _fields_ = [(n, _ct.c_int64) for n in
                ("batch", "prompt_len", "gen_len", "layers", "kv_heads", "head_dim")]


class _Report(_ct.Structure):
    _fields_ = [("decode_steps", _ct.c_int64), ("tokens_per_sec", _ct.c_double),
                ("p50_ms", _ct.c_double), ("p90_ms", _ct.c_double), ("p99_ms", _ct.c_double),
                ("peak_cache_bytes", _ct.c_uint64), ("output_checksum", _ct.c_double),
                ("output_abs_sum", _ct.c_double), ("decode_seconds", _ct.c_double),
                ("n_devices", _ct.c_int32)]


def run_decode_benchmark_native(spec: WorkloadSpec, cfg: CacheConfig, seed: int = 0,
                                devices=(0,), data=None,
                                budget_bytes: int | None = None) -> BenchReport:
    """The reference's run_decode_benchmark (workload.cpp:145-271) in the C++ driver
    (kivi_run_decode_benchmark): one host thread per entry of `devices`, the batch split
    into contiguous blocks, fused tensor-core projection + append and one attend per
    layer and step.  data: optional host (weights [layers, 3, hidden, hidden], prompts
    [batch, prompt_len, hidden], tokens [gen_len, batch, hidden]) fp32 arrays; without
    it the driver draws N(0, 1) data on the devices from `seed` (its own generator, so
    checksums match run_decode_benchmark only for the same `data`)."""
    import numpy as np
    from . import _ERRORS, KiviError
    spec.validate()
    keep = []
    ptrs = [None, None, None]
    if data is not None:
        for i, a in enumerate(data):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
            keep.append(a)
            ptrs[i] = a.ctypes.data
    dev = (_ct.c_int32 * len(devices))(*devices)
    sp = _Spec(spec.batch, spec.prompt_len, spec.gen_len, spec.layers, spec.kv_heads,
               spec.head_dim)
    c = cfg._c()
    rep = _Report()
    L = driver_lib()
    st = L.kivi_run_decode_benchmark(_ct.byref(sp), _ct.addressof(c), dev, len(devices),
                                     int(seed) & (2 ** 64 - 1), ptrs[0], ptrs[1], ptrs[2],
                                     int(budget_bytes or 0), _ct.byref(rep))
    if st != 0:
        msg = L.kivi_driver_last_error().decode(errors="replace")
        if st == 6 and "budget" in msg:
            raise BudgetError(msg)
        raise _ERRORS.get(st, KiviError)(msg)
    return BenchReport(mode="kivi", decode_steps=rep.decode_steps,
                       tokens_per_sec=rep.tokens_per_sec, p50_ms=rep.p50_ms, p90_ms=rep.p90_ms,
                       p99_ms=rep.p99_ms, peak_cache_bytes=rep.peak_cache_bytes,
                       output_checksum=rep.output_checksum, output_abs_sum=rep.output_abs_sum)
