"""Generates tests/golden/kivi_golden.npz by running the REFERENCE itself
(oracle/_ref/ref_cbridge.so: /root/reference/proj/src/{quantize,kv_cache,
attention}.cpp compiled by oracle/Makefile).  Run here, where /root/reference
exists:

    make -C oracle && python tests/golden/make_golden.py

Inputs come from a counter-based generator (splitmix64, reimplemented below
in numpy and in oracle/kivi_oracle.c:oracle_uniform) so every case can be
regenerated bit-identically anywhere.  The fixture is small (< 1 MB).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import Ref  # noqa: E402

M64 = (1 << 64) - 1


def splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def uniform(n, seed, first=0):
    """Exactly oracle_fill_uniform: 24 random bits -> [-1, 1) in fp32."""
    out = np.empty(n, np.float32)
    s = (seed * 0xD1B54A32D192ED03) & M64
    for i in range(n):
        h = splitmix64(s ^ splitmix64(first + i))
        out[i] = np.float32(h >> 40) * np.float32(1.0 / 16777216.0) * np.float32(2.0) - np.float32(1.0)
    return out


TRACES = [  # (bits, G, R, d, l0, steps, seed)
    (2, 4, 8, 8, 13, 20, 1),
    (2, 32, 128, 128, 300, 3, 2),
    (4, 8, 16, 32, 40, 10, 3),
    (1, 4, 8, 12, 9, 9, 4),
    (8, 4, 8, 4, 3, 12, 5),
    (2, 2, 2, 2, 1, 7, 6),
]


def main():
    if not Ref.available():
        raise SystemExit("build oracle/_ref first (make -C oracle)")
    ref = Ref()
    out = {}
    manifest = {"generator": "oracle/_ref (reference compiled from /root/reference)",
                "traces": [], "groups": 0, "matrices": []}

    # 1. quantize_group known answers (reference test_quantize.cpp:42-75) + random
    groups = [np.array(v, np.float32) for v in ([0, 1, 2, 3], [1, 1, 1], [0.0, 0.1, 0.9, 1.0],
                                                [0.0, -0.0], [-0.0, 0.0, 0.5], [2.5])]
    rng = np.random.default_rng(7)
    for n in (1, 2, 3, 4, 16, 32):
        for _ in range(8):
            g = uniform(n, 1000 + len(groups)) * np.float32(5.0)
            if n > 2 and rng.random() < 0.3:
                g[rng.integers(0, n)] = g[0]  # ties
            groups.append(g)
    gi = 0
    for bits in (1, 2, 4, 8):
        for g in groups:
            codes, z, s = ref.quantize_group(g, bits)
            out[f"g{gi}_in"] = g
            out[f"g{gi}_codes"] = codes.astype(np.uint8)
            out[f"g{gi}_zs"] = np.array([z, s], np.float64)
            out[f"g{gi}_bits"] = np.array([bits], np.int32)
            gi += 1
    manifest["groups"] = gi

    # 2. pack bytes
    for bits in (1, 2, 4, 8):
        codes = (np.arange(37, dtype=np.int64) * 7 % (1 << bits)).astype(np.uint8)
        out[f"pack{bits}_codes"] = codes
        out[f"pack{bits}_bytes"] = ref.pack_codes(codes, bits)

    # 3. matrix quantization, both axes
    for mi, (rows, cols, bits, G, pc) in enumerate([(8, 4, 2, 4, 1), (64, 16, 2, 32, 1),
                                                    (3, 64, 2, 32, 0), (12, 6, 4, 4, 1),
                                                    (5, 8, 8, 4, 0), (32, 8, 1, 8, 1)]):
        m = uniform(rows * cols, 2000 + mi).reshape(rows, cols) * np.float32(3.0)
        p, z, s = ref.quantize_matrix(m, bits, G, pc)
        out[f"m{mi}_in"] = m
        out[f"m{mi}_packed"], out[f"m{mi}_z"], out[f"m{mi}_s"] = p, z, s
        manifest["matrices"].append([rows, cols, bits, G, pc])

    # 4. streaming cache traces: prefill l0 tokens, then `steps` decode_attention
    for ti, (bits, G, R, d, l0, steps, seed) in enumerate(TRACES):
        n = l0 + steps
        K = uniform(n * d, seed * 10 + 1).reshape(n, d)
        V = uniform(n * d, seed * 10 + 2).reshape(n, d)
        Q = uniform(steps * d, seed * 10 + 3).reshape(steps, d)
        u = ref.unit(bits, G, R, d)
        u.prefill(K[:l0], V[:l0])
        outs = np.zeros((steps, d), np.float32)
        w_last = None
        for s_ in range(steps):
            o, w = u.decode(Q[s_], K[l0 + s_], V[l0 + s_], weights=True)
            outs[s_] = o
            w_last = w
        st = u.export()
        c = u.counters()
        pre = f"t{ti}_"
        out[pre + "K"], out[pre + "V"], out[pre + "Q"] = K, V, Q
        out[pre + "out"] = outs
        out[pre + "w_last"] = w_last
        for k, v in st.items():
            out[pre + k] = v
        out[pre + "counters"] = np.array([c["key_grouped"], c["key_residual"], c["total"],
                                          c["key_capacity"], c["value_grouped"],
                                          c["value_residual"], c["value_capacity"],
                                          c["key_memory"], c["value_memory"]], np.int64)
        km, vm = u.materialize()
        out[pre + "mat_k"], out[pre + "mat_v"] = km, vm
        manifest["traces"].append([bits, G, R, d, l0, steps, seed])

    # 5. reference_attention
    q = uniform(2 * 16, 91).reshape(2, 16)
    K = uniform(37 * 16, 92).reshape(37, 16)
    V = uniform(37 * 16, 93).reshape(37, 16)
    out["ra_q"], out["ra_K"], out["ra_V"] = q, K, V
    out["ra_out"] = ref.reference_attention(q, K, V)

    np.savez_compressed(os.path.join(HERE, "kivi_golden.npz"), **out)
    with open(os.path.join(HERE, "kivi_golden.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
