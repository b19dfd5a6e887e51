"""TEST INFRASTRUCTURE: ctypes wrappers over the two CPU checkers.

* ``Port`` — oracle/liboracle.so, this repo's plain-C restatement of the
  reference hot path (oracle/kivi_oracle.c).
* ``Ref``  — oracle/_ref/ref_cbridge.so, the REFERENCE itself compiled from
  /root/reference by oracle/Makefile (prebuilt files travel to the GPU box).

Both expose the same interface so a parity test can run against either.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_LIB = os.path.join(ROOT, "oracle", "liboracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "ref_cbridge.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64


def _p(a):
    return None if a is None else a.ctypes.data


class CheckerError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"code {code}: {msg}")
        self.code = code  # 1 shape, 2 usage, 3 config


class _Base:
    def uniform(self, n, seed, first=0):
        out = np.empty((n,), np.float32)
        self._port().oracle_fill_uniform(out.ctypes.data, n, ctypes.c_uint64(seed),
                                         ctypes.c_uint64(first))
        return out

    @staticmethod
    def _port():
        return Port.lib()


class Port(_Base):
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(PORT_LIB)
            sig = {
                "oracle_quantize_group": (ctypes.c_int, [P, I64, ctypes.c_int, P, P, P]),
                "oracle_dequantize_group": (None, [P, I64, ctypes.c_double, ctypes.c_double, P]),
                "oracle_pack_codes": (ctypes.c_int, [P, I64, ctypes.c_int, P]),
                "oracle_unpack_codes": (ctypes.c_int, [P, I64, I64, ctypes.c_int, P]),
                "oracle_quantize_matrix": (ctypes.c_int,
                                           [P, I64, I64, ctypes.c_int, I64, ctypes.c_int, P, P, P]),
                "oracle_dequantize_matrix": (None, [P, P, P, I64, I64, ctypes.c_int, I64,
                                                    ctypes.c_int, P]),
                "oracle_unit_new": (P, [ctypes.c_int, I64, I64, I64]),
                "oracle_unit_free": (None, [P]),
                "oracle_prefill": (ctypes.c_int, [P, P, P, I64]),
                "oracle_append": (None, [P, P, P]),
                "oracle_decode": (None, [P, P, P, P, ctypes.c_int, P, P]),
                "oracle_attend": (None, [P, P, ctypes.c_int, P, P]),
                "oracle_materialize": (None, [P, P, P]),
                "oracle_reference_attention": (None, [P, I64, P, P, I64, I64, ctypes.c_int, P]),
                "oracle_counters": (None, [P, P]),
                "oracle_fill_uniform": (None, [P, I64, ctypes.c_uint64, ctypes.c_uint64]),
                "oracle_uniform": (ctypes.c_float, [ctypes.c_uint64, ctypes.c_uint64]),
            }
            for n in ("key_packed", "value_packed"):
                sig[f"oracle_{n}"] = (P, [P, P])
            for n in ("key_zero", "key_scale", "value_zero", "value_scale"):
                sig[f"oracle_{n}"] = (P, [P, P])
            for n in ("key_residual", "value_residual"):
                sig[f"oracle_{n}"] = (P, [P, P])
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            cls._lib = L
        return cls._lib

    name = "port"

    def quantize_group(self, v, bits):
        v = np.ascontiguousarray(v, np.float32)
        codes = np.zeros((max(v.size, 1),), np.uint8)
        z, s = ctypes.c_double(), ctypes.c_double()
        rc = self.lib().oracle_quantize_group(_p(v), v.size, bits, _p(codes), ctypes.byref(z),
                                              ctypes.byref(s))
        if rc:
            raise CheckerError(rc)
        return codes[:v.size], z.value, s.value

    def pack_codes(self, codes, bits):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(((codes.size * bits + 7) // 8 + 1,), np.uint8)
        rc = self.lib().oracle_pack_codes(_p(codes), codes.size, bits, _p(out))
        if rc:
            raise CheckerError(rc)
        return out[:(codes.size * bits + 7) // 8]

    def quantize_matrix(self, m, bits, G, per_channel):
        m = np.ascontiguousarray(m, np.float32)
        r, c = m.shape
        packed = np.zeros(((r * c * bits + 7) // 8 + 1,), np.uint8)
        ng = r * c // G
        z = np.zeros((max(ng, 1),), np.float64)
        s = np.zeros((max(ng, 1),), np.float64)
        rc = self.lib().oracle_quantize_matrix(_p(m), r, c, bits, G, int(per_channel), _p(packed),
                                               _p(z), _p(s))
        if rc:
            raise CheckerError(rc)
        return packed[:(r * c * bits + 7) // 8], z[:ng], s[:ng]

    def reference_attention(self, q, K, V, scale_logits=True):
        q, K, V = (np.ascontiguousarray(a, np.float32) for a in (q, K, V))
        out = np.zeros((q.shape[0], q.shape[1]), np.float32)
        self.lib().oracle_reference_attention(_p(q), q.shape[0], _p(K), _p(V), K.shape[0],
                                              K.shape[1], int(scale_logits), _p(out))
        return out

    def unit(self, bits, G, R, d):
        return PortUnit(self.lib(), bits, G, R, d)


class PortUnit:
    def __init__(self, L, bits, G, R, d):
        self.L, self.d = L, d
        self.h = L.oracle_unit_new(bits, G, R, d)

    def __del__(self):
        try:
            self.L.oracle_unit_free(self.h)
        except Exception:
            pass

    def prefill(self, K, V):
        K, V = np.ascontiguousarray(K, np.float32), np.ascontiguousarray(V, np.float32)
        rc = self.L.oracle_prefill(self.h, _p(K), _p(V), K.shape[0])
        if rc:
            raise CheckerError(rc)

    def append(self, tk, tv):
        tk, tv = np.ascontiguousarray(tk, np.float32), np.ascontiguousarray(tv, np.float32)
        self.L.oracle_append(self.h, _p(tk), _p(tv))

    def decode(self, q, tk, tv, scale_logits=True, weights=False):
        q, tk, tv = (np.ascontiguousarray(a, np.float32) for a in (q, tk, tv))
        out = np.zeros((self.d,), np.float32)
        self.append(tk, tv)
        w = np.zeros((self.counters()["total"],), np.float32) if weights else None
        self.L.oracle_attend(self.h, _p(q), int(scale_logits), _p(out), _p(w))
        return (out, w) if weights else out

    def counters(self):
        o = np.zeros((9,), np.int64)
        self.L.oracle_counters(self.h, _p(o))
        return {"key_grouped": o[0], "key_residual": o[1], "total": o[2], "key_capacity": o[3],
                "value_grouped": o[4], "value_residual": o[5], "value_capacity": o[6],
                "key_memory": o[7], "value_memory": o[8]}

    def export(self):
        L, h, d = self.L, self.h, self.d
        n = ctypes.c_int64()

        def arr(fn, dtype, count_fn=None):
            ptr = fn(h, ctypes.byref(n))
            cnt = n.value
            if cnt == 0:
                return np.zeros((0,), dtype)
            return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(
                np.ctypeslib.as_ctypes_type(dtype))), shape=(cnt,)).copy()

        out = {
            "key_packed": arr(L.oracle_key_packed, np.uint8),
            "key_zero": arr(L.oracle_key_zero, np.float64),
            "key_scale": arr(L.oracle_key_scale, np.float64),
            "value_packed": arr(L.oracle_value_packed, np.uint8),
            "value_zero": arr(L.oracle_value_zero, np.float64),
            "value_scale": arr(L.oracle_value_scale, np.float64),
        }
        for k, fn in (("key_residual", L.oracle_key_residual),
                      ("value_residual", L.oracle_value_residual)):
            ptr = fn(h, ctypes.byref(n))
            rows = n.value
            if rows == 0:
                out[k] = np.zeros((0, d), np.float32)
            else:
                out[k] = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_float)),
                                               shape=(rows * d,)).reshape(rows, d).copy()
        return out

    def materialize(self):
        l = int(self.counters()["total"])
        k = np.zeros((l, self.d), np.float32)
        v = np.zeros((l, self.d), np.float32)
        self.L.oracle_materialize(self.h, _p(k), _p(v))
        return k, v


class Ref(_Base):
    """The reference library itself (oracle/_ref)."""
    _lib = None
    name = "ref"

    @classmethod
    def available(cls):
        return os.path.exists(REF_LIB)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(REF_LIB)
            CI = ctypes.c_int
            sig = {
                "ref_last_error": (ctypes.c_char_p, []),
                "ref_state_new": (P, []),
                "ref_state_free": (None, [P]),
                "ref_state_clone": (P, [P]),
                "ref_prefill": (CI, [P, CI, I64, I64, I64, P, P, I64]),
                "ref_append": (CI, [P, CI, I64, I64, I64, P, P]),
                "ref_decode": (CI, [P, CI, I64, I64, I64, P, P, P, CI, P, P]),
                "ref_counters": (CI, [P, P, P]),
                "ref_export": (CI, [P, P, P, P, P, P, P, P, P]),
                "ref_materialize": (CI, [P, P, P]),
                "ref_quantize_group": (CI, [P, I64, CI, P, P, P]),
                "ref_pack_codes": (CI, [P, I64, CI, P]),
                "ref_quantize_matrix": (CI, [P, I64, I64, CI, I64, CI, P, P, P]),
                "ref_reference_attention": (CI, [P, I64, P, P, I64, I64, CI, P]),
                "ref_bench_decode": (CI, [CI, I64, I64, I64, I64, I64, I64, I64, CI,
                                          ctypes.c_uint64, P, P]),
                "ref_estimate_memory": (CI, [P, CI, I64, I64, P, P]),
                "ref_max_batch_at_budget": (CI, [P, ctypes.c_uint64, CI, CI, I64, I64, P]),
                "ref_workload_data": (CI, [P, ctypes.c_uint64, P, P, P]),
                "ref_run_decode_benchmark": (CI, [P, ctypes.c_uint64, CI, CI, I64, I64,
                                                  ctypes.c_uint64, P, P]),
                "ref_write_dump": (CI, [ctypes.c_char_p, P, I64, I64, I64]),
                "ref_read_dump": (CI, [ctypes.c_char_p, P, P, P]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            cls._lib = L
        return cls._lib

    def _chk(self, rc):
        if rc:
            raise CheckerError(rc, self.lib().ref_last_error().decode())

    def quantize_group(self, v, bits):
        v = np.ascontiguousarray(v, np.float32)
        codes = np.zeros((max(v.size, 1),), np.uint8)
        z, s = ctypes.c_double(), ctypes.c_double()
        self._chk(self.lib().ref_quantize_group(_p(v), v.size, bits, _p(codes), ctypes.byref(z),
                                                ctypes.byref(s)))
        return codes[:v.size], z.value, s.value

    def pack_codes(self, codes, bits):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(((codes.size * bits + 7) // 8 + 1,), np.uint8)
        self._chk(self.lib().ref_pack_codes(_p(codes), codes.size, bits, _p(out)))
        return out[:(codes.size * bits + 7) // 8]

    def quantize_matrix(self, m, bits, G, per_channel):
        m = np.ascontiguousarray(m, np.float32)
        r, c = m.shape
        packed = np.zeros(((r * c * bits + 7) // 8 + 1,), np.uint8)
        ng = r * c // G
        z = np.zeros((max(ng, 1),), np.float64)
        s = np.zeros((max(ng, 1),), np.float64)
        self._chk(self.lib().ref_quantize_matrix(_p(m), r, c, bits, G, int(per_channel),
                                                 _p(packed), _p(z), _p(s)))
        return packed[:(r * c * bits + 7) // 8], z[:ng], s[:ng]

    def reference_attention(self, q, K, V, scale_logits=True):
        q, K, V = (np.ascontiguousarray(a, np.float32) for a in (q, K, V))
        out = np.zeros((q.shape[0], q.shape[1]), np.float32)
        self._chk(self.lib().ref_reference_attention(_p(q), q.shape[0], _p(K), _p(V), K.shape[0],
                                                     K.shape[1], int(scale_logits), _p(out)))
        return out

    def unit(self, bits, G, R, d):
        return RefUnit(self, bits, G, R, d)

    # ---- workload layer (reference workload.cpp) --------------------------
    @staticmethod
    def _spec(spec):
        return np.array([spec.batch, spec.prompt_len, spec.gen_len, spec.layers, spec.kv_heads,
                         spec.head_dim], np.int64)

    def estimate_memory(self, spec, bits, G, R):
        sp = self._spec(spec)
        out = np.zeros(5, np.uint64)
        ratio = ctypes.c_double()
        self._chk(self.lib().ref_estimate_memory(_p(sp), bits, G, R, _p(out), ctypes.byref(ratio)))
        return dict(zip(["fp_bytes", "kivi_bytes", "code_bytes", "scale_zero_bytes",
                         "residual_bytes"], (int(x) for x in out)), compression_ratio=ratio.value)

    def max_batch_at_budget(self, spec, budget, fp_mode, bits, G, R):
        sp = self._spec(spec)
        out = ctypes.c_int64()
        self._chk(self.lib().ref_max_batch_at_budget(_p(sp), budget, int(fp_mode), bits, G, R,
                                                     ctypes.byref(out)))
        return out.value

    def workload_data(self, spec, seed):
        """The exact weights / prompts / decode tokens run_decode_benchmark draws."""
        sp = self._spec(spec)
        hid = spec.head_dim * spec.kv_heads
        w = np.zeros((spec.layers, 3, hid, hid), np.float32)
        pr = np.zeros((spec.batch, spec.prompt_len, hid), np.float32)
        tk = np.zeros((max(spec.gen_len, 1), spec.batch, hid), np.float32)
        self._chk(self.lib().ref_workload_data(_p(sp), seed, _p(w), _p(pr), _p(tk)))
        return w, pr, tk[:spec.gen_len]

    def run_decode_benchmark(self, spec, seed, fp_mode, bits, G, R, budget=0):
        sp = self._spec(spec)
        out = np.zeros(2, np.float64)
        peak = ctypes.c_uint64()
        self._chk(self.lib().ref_run_decode_benchmark(_p(sp), seed, int(fp_mode), bits, G, R,
                                                      budget, _p(out), ctypes.byref(peak)))
        return {"tokens_per_sec": float(out[0]), "output_checksum": float(out[1]),
                "peak_cache_bytes": int(peak.value)}

    # ---- KVQD dumps (reference dump_io.cpp) ---------------------------------
    def write_dump(self, path, tensors):
        t = np.ascontiguousarray(np.stack([np.asarray(x, np.float32) for x in tensors]))
        self._chk(self.lib().ref_write_dump(path.encode(), _p(t), t.shape[0], t.shape[1],
                                            t.shape[2]))

    def read_dump(self, path):
        """-> (list of arrays, None) or (None, (code, byte_offset or None))."""
        dims = np.zeros(3, np.int64)
        off = ctypes.c_uint64()
        rc = self.lib().ref_read_dump(path.encode(), _p(dims), None, ctypes.byref(off))
        if rc:
            return None, (rc, off.value if rc == 5 else None)
        data = np.zeros(int(dims.prod()), np.float32)
        self._chk(self.lib().ref_read_dump(path.encode(), _p(dims), _p(data), ctypes.byref(off)))
        return list(data.reshape(dims)), None

    def bench_decode(self, bits, G, R, d, n_units, l_prefill, warmup, steps, threads, seed=1):
        secs, cs = ctypes.c_double(), ctypes.c_double()
        self._chk(self.lib().ref_bench_decode(bits, G, R, d, n_units, l_prefill, warmup, steps,
                                              threads, seed, ctypes.byref(secs),
                                              ctypes.byref(cs)))
        return secs.value, cs.value


class RefUnit:
    def __init__(self, ref, bits, G, R, d):
        self.ref, self.L = ref, ref.lib()
        self.cfg = (bits, G, R, d)
        self.d = d
        self.h = self.L.ref_state_new()

    def __del__(self):
        try:
            self.L.ref_state_free(self.h)
        except Exception:
            pass

    def prefill(self, K, V):
        K, V = np.ascontiguousarray(K, np.float32), np.ascontiguousarray(V, np.float32)
        self.ref._chk(self.L.ref_prefill(self.h, *self.cfg, _p(K), _p(V), K.shape[0]))

    def clone(self):
        """Deep copy of the state (the reference's states are copyable,
        workload.cpp:166-167): one prefill serves several query heads."""
        c = RefUnit.__new__(RefUnit)
        c.ref, c.L, c.cfg, c.d = self.ref, self.L, self.cfg, self.d
        c.h = self.L.ref_state_clone(self.h)
        return c

    def append(self, tk, tv):
        tk, tv = np.ascontiguousarray(tk, np.float32), np.ascontiguousarray(tv, np.float32)
        self.ref._chk(self.L.ref_append(self.h, *self.cfg, _p(tk), _p(tv)))

    def decode(self, q, tk, tv, scale_logits=True, weights=False):
        q, tk, tv = (np.ascontiguousarray(a, np.float32) for a in (q, tk, tv))
        out = np.zeros((self.d,), np.float32)
        w = np.zeros((self.counters()["total"] + 1,), np.float32) if weights else None
        self.ref._chk(self.L.ref_decode(self.h, *self.cfg, _p(q), _p(tk), _p(tv),
                                        int(scale_logits), _p(out), _p(w)))
        return (out, w) if weights else out

    def counters(self):
        c = np.zeros((8,), np.int64)
        s = np.zeros((6,), np.uint64)
        self.ref._chk(self.L.ref_counters(self.h, _p(c), _p(s)))
        return {"key_grouped": c[0], "key_residual": c[1], "total": c[2], "key_capacity": c[3],
                "value_grouped": c[4], "value_residual": c[5], "value_capacity": c[7],
                "key_memory": int(s[4]), "value_memory": int(s[5]),
                "key_packed_bytes": int(s[0]), "key_groups": int(s[1]),
                "value_packed_bytes": int(s[2]), "value_groups": int(s[3])}

    def export(self):
        c = self.counters()
        d = self.d
        out = {
            "key_packed": np.zeros((c["key_packed_bytes"],), np.uint8),
            "key_zero": np.zeros((c["key_groups"],), np.float64),
            "key_scale": np.zeros((c["key_groups"],), np.float64),
            "key_residual": np.zeros((int(c["key_residual"]), d), np.float32),
            "value_packed": np.zeros((c["value_packed_bytes"],), np.uint8),
            "value_zero": np.zeros((c["value_groups"],), np.float64),
            "value_scale": np.zeros((c["value_groups"],), np.float64),
            "value_residual": np.zeros((int(c["value_residual"]), d), np.float32),
        }
        self.ref._chk(self.L.ref_export(self.h, *[_p(out[k]) if out[k].size else None for k in (
            "key_packed", "key_zero", "key_scale", "key_residual", "value_packed", "value_zero",
            "value_scale", "value_residual")]))
        return out

    def materialize(self):
        l = int(self.counters()["total"])
        k = np.zeros((l, self.d), np.float32)
        v = np.zeros((l, self.d), np.float32)
        self.ref._chk(self.L.ref_materialize(self.h, _p(k), _p(v)))
        return k, v


def checkers():
    """The checkers available here: always the port; the reference when built."""
    out = [Port()]
    if Ref.available():
        out.append(Ref())
    return out


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
