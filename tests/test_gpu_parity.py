"""GPU parity: the CUDA path (through the C-ABI) against the reference.

The checker is the reference itself (oracle/_ref, compiled from its own
sources) when present, else the plain-C port (oracle/liboracle.so).
Bars:
  * packed codes, zero-points, scales, residual rows, counters and
    materialised K/V: bit-exact;
  * decode outputs, generic kernel (reference arithmetic order): rel-L2 <= 1e-6;
  * decode outputs, fast sm_100a kernel (fp32 FFMA2 accumulation):
    rel-L2 <= 1e-5 (the reference's own hybrid bound, test_attention.cpp:79);
  * softmax weights: max |diff| <= 1e-6 (generic), <= 1e-5 (fast).
"""
import os

import numpy as np
import pytest

from oracles import Port, Ref, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
kb = pytest.importorskip("paper_2402_02750_b200")


def checker():
    return Ref() if Ref.available() else Port()


def rnd(rng, *shape, scale=1.0):
    return rng.uniform(-scale, scale, size=shape).astype(np.float32)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_state_equal(got, want, where=""):
    for k in ("key_packed", "key_zero", "key_scale", "key_residual", "value_packed",
              "value_zero", "value_scale", "value_residual"):
        g, w = np.asarray(got[k]), np.asarray(want[k])
        assert g.shape == w.shape, f"{where} {k}: shape {g.shape} != {w.shape}"
        assert g.tobytes() == w.tobytes(), f"{where} {k}: not bit-identical"


def assert_counters(cache, unit_ref, where=""):
    i = cache.info()
    c = unit_ref.counters()
    assert i["total_tokens"] == c["total"], where
    assert i["key_grouped_tokens"] == c["key_grouped"], where
    assert i["key_residual_rows"] == c["key_residual"], where
    assert i["key_residual_capacity"] == c["key_capacity"], where
    assert i["value_grouped_tokens"] == c["value_grouped"], where
    assert i["value_residual_rows"] == c["value_residual"], where
    assert i["value_residual_capacity"] == c["value_capacity"], where
    assert i["key_memory_bytes"] == c["key_memory"], where
    assert i["value_memory_bytes"] == c["value_memory"], where


# (bits, G, R, d) — the reference tests' shapes plus the headline shape.
STATE_CONFIGS = [
    (2, 32, 128, 128), (4, 32, 128, 128), (8, 32, 128, 128), (1, 32, 64, 64),
    (2, 4, 8, 8), (2, 8, 16, 32), (8, 4, 8, 4), (2, 2, 2, 2), (2, 2, 4, 2), (4, 2, 4, 2),
    (2, 16, 32, 64), (1, 4, 8, 12), (4, 4, 8, 4), (2, 32, 512, 32),
]


# ---------------------------------------------------------------- quantizer --
@pytest.mark.parametrize("bits", [1, 2, 4, 8])
@pytest.mark.parametrize("G,per_channel", [(32, True), (32, False), (4, True), (2, False),
                                           (3, True), (16, False)])
def test_quantize_matrix_bit_exact(cuda, bits, G, per_channel):
    ck = checker()
    rng = np.random.default_rng(100 + bits * 7 + G)
    rows, cols = (G * 6, 10) if per_channel else (9, G * 5)
    m = rnd(rng, rows, cols, scale=3.0)
    # degenerate / tie-heavy groups: constants, repeated values, +-0
    m[:G, 0] = 1.25
    m[:, 1] = np.round(m[:, 1] * 2) / 2
    m[0, 2], m[1, 2] = 0.0, -0.0
    p, z, s = kb.quantize_matrix(dev(m), bits, G, per_channel)
    rp, rz, rs = ck.quantize_matrix(m, bits, G, per_channel)
    assert p.cpu().numpy().tobytes() == rp.tobytes()
    assert z.cpu().numpy().tobytes() == rz.tobytes()
    assert s.cpu().numpy().tobytes() == rs.tobytes()
    back = kb.dequantize_matrix(p, z, s, rows, cols, bits, G, per_channel).cpu().numpy()
    want = np.zeros_like(m)
    Port.lib().oracle_dequantize_matrix(rp.ctypes.data, rz.ctypes.data, rs.ctypes.data, rows,
                                        cols, bits, G, int(per_channel), want.ctypes.data)
    assert back.tobytes() == want.tobytes()


def test_quantize_group_spec_examples(cuda):
    # reference test_quantize.cpp:42-75 through the device quantizer
    cases = [([0, 1, 2, 3], [0, 1, 2, 3], 0.0, 1.0), ([1, 1, 1], [0, 0, 0], 1.0, 1.0),
             ([0.0, 0.1, 0.9, 1.0], [0, 0, 3, 3], 0.0, 1.0 / 3.0)]
    for vals, codes, z0, s0 in cases:
        m = np.array([vals], np.float32)
        p, z, s = kb.quantize_matrix(dev(m), 2, len(vals), False)
        got = kb.unpack_codes(p, len(vals), 2).cpu().numpy().tolist()
        assert got == codes
        assert z.cpu().item() == z0
        assert abs(s.cpu().item() - s0) < 1e-15
    # pack examples (test_quantize.cpp:100-108)
    assert kb.pack_codes(dev(np.array([0, 1, 2, 3], np.uint8)), 2).cpu().tolist() == [0xE4]
    assert kb.pack_codes(dev(np.array([3], np.uint8)), 2).cpu().tolist() == [0x03]
    assert kb.pack_codes(dev(np.array([0xA, 0xB], np.uint8)), 4).cpu().tolist() == [0xBA]
    with pytest.raises(kb.UsageError):
        kb.pack_codes(dev(np.array([4], np.uint8)), 2)
    with pytest.raises(kb.UsageError):
        kb.pack_codes(dev(np.array([1], np.uint8)), 3)
    with pytest.raises(kb.ShapeError):
        kb.quantize_matrix(dev(rnd(np.random.default_rng(0), 5, 2)), 2, 2, True)
    with pytest.raises(kb.ConfigError):
        kb.quantize_matrix(dev(rnd(np.random.default_rng(0), 4, 2)), 3, 2, True)


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 8])
def test_quantize_group_single_launch(cuda, bits):
    """kivi_quantize_group (the facade's quantize_group: one launch that also
    dequantizes) == the reference's quantize_group + dequantize_group, on group
    sizes 1..1000 with ties, constants and signed zeros."""
    import ctypes
    from oracles import Port
    rng = np.random.default_rng(50 + bits)
    cases = [rnd(rng, n) for n in (1, 2, 3, 31, 32, 33, 255, 256, 257, 1000)]
    cases += [np.full(17, 0.1, np.float32), np.array([0.0, -0.0, 0.5, -0.0], np.float32),
              np.array([-0.5, -0.0, 0.0, -0.5], np.float32),
              np.round(rnd(rng, 64) * 2) / 2]
    lib = kb.lib()
    port = Port.lib()
    for v in cases:
        v = np.ascontiguousarray(v, np.float32)
        n = v.size
        dv = dev(v)
        codes = torch.empty(n, dtype=torch.uint8, device="cuda")
        zs = torch.empty(2, dtype=torch.float64, device="cuda")
        deq = torch.empty(n, dtype=torch.float32, device="cuda")
        st = lib.kivi_quantize_group(dv.data_ptr(), n, bits, codes.data_ptr(), zs.data_ptr(),
                                     zs.data_ptr() + 8, deq.data_ptr(), None)
        assert st == 0, lib.kivi_last_error()
        torch.cuda.synchronize()
        want_c = np.zeros(n, np.uint8)
        want_zs = np.zeros(2, np.float64)
        port.oracle_quantize_group(v.ctypes.data, n, bits, want_c.ctypes.data,
                                   want_zs.ctypes.data, want_zs[1:].ctypes.data)
        want_d = np.zeros(n, np.float32)
        port.oracle_dequantize_group(want_c.ctypes.data, n, ctypes.c_double(want_zs[0]),
                                     ctypes.c_double(want_zs[1]), want_d.ctypes.data)
        assert codes.cpu().numpy().tobytes() == want_c.tobytes(), (bits, n)
        assert zs.cpu().numpy().tobytes() == want_zs.tobytes(), (bits, n)
        assert deq.cpu().numpy().tobytes() == want_d.tobytes(), (bits, n)
    assert lib.kivi_quantize_group(dv.data_ptr(), 0, bits, codes.data_ptr(), zs.data_ptr(),
                                   zs.data_ptr() + 8, None, None) == 2  # KIVI_ERR_USAGE


def test_pack_unpack_identity(cuda):
    rng = np.random.default_rng(12)
    for bits in (1, 2, 4, 8):
        for n in (1, 7, 1000, 10001):
            codes = rng.integers(0, 1 << bits, size=n, dtype=np.uint8)
            p = kb.pack_codes(dev(codes), bits)
            assert p.cpu().numpy().tobytes() == Port().pack_codes(codes, bits).tobytes()
            assert kb.unpack_codes(p, n, bits).cpu().numpy().tobytes() == codes.tobytes()


# ------------------------------------------------------------ cache state ----
@pytest.mark.parametrize("cfg", STATE_CONFIGS)
def test_prefill_then_stream_state_bit_exact(cuda, cfg):
    bits, G, R, d = cfg
    ck = checker()
    rng = np.random.default_rng(hash(cfg) % 2**32)
    U = 3
    n = 3 * R + 7
    K = rnd(rng, U, n, d)
    V = rnd(rng, U, n, d)
    K[1, :G, :] = 0.5  # constant key groups in unit 1
    k0 = max(1, R // 2 + 3)
    cache = kb.KVCache(kb.CacheConfig(bits, G, R, d), U)
    cache.prefill(dev(K[:, :k0]), dev(V[:, :k0]))
    refs = [ck.unit(bits, G, R, d) for _ in range(U)]
    for u in range(U):
        refs[u].prefill(K[u, :k0], V[u, :k0])
    for t in range(k0, n + 1):
        if t in (k0, k0 + 1, R, R + 1, 2 * R - 1, 2 * R, n):
            torch.cuda.synchronize()
            for u in range(U):
                assert_state_equal(cache.export_unit(u), refs[u].export(), f"cfg={cfg} t={t} u={u}")
                assert_counters(cache, refs[u], f"cfg={cfg} t={t}")
            km, vm = cache.materialize()
            for u in range(U):
                rk, rv = refs[u].materialize()
                assert km[u].cpu().numpy().tobytes() == rk.tobytes()
                assert vm[u].cpu().numpy().tobytes() == rv.tobytes()
        if t == n:
            break
        cache.append(dev(K[:, t]), dev(V[:, t]))
        for u in range(U):
            refs[u].append(K[u, t], V[u, t])


@pytest.mark.parametrize("bits", [2, 4])
def test_fast_quantizer_signed_zero_and_tie_groups(cuda, bits):
    """The d = 128, G = 32 kernels (prefill, warp-per-unit append with its
    value pop, parallel key flush) decide codes in fp32 via the magic-number
    rint and take min / max with FMNMX: groups whose extreme is +0 / -0 in
    both orders, exact rounding ties (x = k + 1/2: the exact double path) and
    all-zero groups of mixed sign must still give the reference's state."""
    ck = checker()
    rng = np.random.default_rng(77 + bits)
    U, d, R, G = 4, 128, 128, 32
    n = 3 * R + 40
    pools = [np.array([-0.0, 0.0, 0.25, 0.75, 1.5], np.float32),   # min is a signed zero
             np.array([-1.5, -0.25, -0.75, -0.0, 0.0], np.float32),  # max is a signed zero
             None,                                                  # random
             np.array([-0.0, 0.0], np.float32)]                      # all-zero groups
    K = np.empty((U, n, d), np.float32)
    V = np.empty((U, n, d), np.float32)
    for u, pool in enumerate(pools):
        if pool is None:
            K[u], V[u] = rnd(rng, n, d), rnd(rng, n, d)
        else:
            K[u], V[u] = rng.choice(pool, (n, d)), rng.choice(pool, (n, d))
    k0 = R + 45
    cache = kb.KVCache(kb.CacheConfig(bits, G, R, d), U)
    cache.prefill(dev(K[:, :k0]), dev(V[:, :k0]))
    refs = [ck.unit(bits, G, R, d) for _ in range(U)]
    for u in range(U):
        refs[u].prefill(K[u, :k0], V[u, :k0])
    for t in range(k0, n + 1):
        if t in (k0, 2 * R, 2 * R + 1, 3 * R, n):
            torch.cuda.synchronize()
            for u in range(U):
                assert_state_equal(cache.export_unit(u), refs[u].export(), f"t={t} u={u}")
        if t == n:
            break
        cache.append(dev(K[:, t]), dev(V[:, t]))
        for u in range(U):
            refs[u].append(K[u, t], V[u, t])
    cache.close()


def test_prefill_unaligned_rows(cuda):
    """Prefill rows that are not 16-byte aligned (a view one float into a
    buffer) take the scalar kernels; the state is the same bit for bit."""
    ck = checker()
    rng = np.random.default_rng(31)
    U, l, d = 2, 300, 128
    K, V = rnd(rng, U, l, d), rnd(rng, U, l, d)
    kbuf = torch.empty(U * l * d + 1, device="cuda")
    vbuf = torch.empty(U * l * d + 1, device="cuda")
    kv = kbuf[1:].view(U, l, d)
    vv = vbuf[1:].view(U, l, d)
    kv.copy_(dev(K))
    vv.copy_(dev(V))
    cache = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    cache.prefill(kv, vv)
    refs = []
    for u in range(U):
        r = ck.unit(2, 32, 128, d)
        r.prefill(K[u], V[u])
        assert_state_equal(cache.export_unit(u), r.export(), f"u={u}")
        refs.append(r)
    # decode with unaligned q / k / v rows: routed to the generic kernels
    for step in range(3):
        q, tk, tv = rnd(rng, U, d), rnd(rng, U, d), rnd(rng, U, d)
        bufs = [torch.empty(U * d + 1, device="cuda") for _ in range(3)]
        qv, tkv, tvv = (b[1:].view(U, d) for b in bufs)
        qv.copy_(dev(q))
        tkv.copy_(dev(tk))
        tvv.copy_(dev(tv))
        out = cache.decode(qv.view(U, 1, d), tkv, tvv).cpu().numpy()
        for u in range(U):
            want = refs[u].decode(q[u], tk[u], tv[u])
            assert rel_l2(out[u, 0], want) <= 1e-6, f"step {step} unit {u}"
    torch.cuda.synchronize()
    for u in range(U):
        assert_state_equal(cache.export_unit(u), refs[u].export(), f"after decode u={u}")
    cache.close()


@pytest.mark.parametrize("bits", [2, 4])
def test_long_stream_many_flushes(cuda, bits, monkeypatch):
    """1,100 appends from l = 301 (9 key flushes, 36 early key-tile quantisations,
    1,100 value pops) on the fast kernels, decoding every step: outputs within
    1e-5 of the reference at every step and the state bit-identical at every
    flush boundary -- no drift between the device store and the reference's."""
    monkeypatch.setenv("KIVI_SMALL_ITEMS", "0")
    ck = checker()
    rng = np.random.default_rng(900 + bits)
    U, d, l0, steps = 4, 128, 301, 1100
    K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
    cache = kb.KVCache(kb.CacheConfig(bits, 32, 128, d), U)
    cache.prefill(dev(K), dev(V))
    refs = [ck.unit(bits, 32, 128, d) for _ in range(U)]
    for u in range(U):
        refs[u].prefill(K[u], V[u])
    worst = 0.0
    for s_ in range(steps):
        q, tk, tv = rnd(rng, U, d), rnd(rng, U, d), rnd(rng, U, d)
        out = cache.decode(dev(q)[:, None, :].contiguous(), dev(tk), dev(tv)).cpu().numpy()
        for u in range(U):
            worst = max(worst, rel_l2(out[u, 0], refs[u].decode(q[u], tk[u], tv[u])))
        if (l0 + s_ + 1) % 128 == 0:
            for u in range(U):
                assert_state_equal(cache.export_unit(u), refs[u].export(), f"l={l0 + s_ + 1} u={u}")
    assert worst <= 1e-5, worst
    cache.close()


def test_streaming_equals_batch(cuda):
    # reference test_kv_cache.cpp:133-157 on the device path
    rng = np.random.default_rng(25)
    for trial in range(10):
        bits, G, R, d = (2, 4, 8, 8)
        n = int(rng.integers(1, 101))
        k = int(rng.integers(1, n + 1))
        K, V = rnd(rng, 1, n, d), rnd(rng, 1, n, d)
        batch = kb.KVCache(kb.CacheConfig(bits, G, R, d), 1)
        batch.prefill(dev(K), dev(V))
        stream = kb.KVCache(kb.CacheConfig(bits, G, R, d), 1)
        stream.prefill(dev(K[:, :k]), dev(V[:, :k]))
        for t in range(k, n):
            stream.append(dev(K[:, t]), dev(V[:, t]))
        assert_state_equal(stream.export_unit(0), batch.export_unit(0), f"trial {trial}")


# ----------------------------------------------------------------- decode ----
def run_decode(cfg, U, l0, steps, path, seed, weights=True, scale=True):
    bits, G, R, d = cfg
    ck = checker()
    rng = np.random.default_rng(seed)
    K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
    cache = kb.KVCache(kb.CacheConfig(bits, G, R, d), U)
    cache.set_attend_path(path)
    cache.prefill(dev(K), dev(V))
    refs = [ck.unit(bits, G, R, d) for _ in range(U)]
    for u in range(U):
        refs[u].prefill(K[u], V[u])
    worst_out, worst_w = 0.0, 0.0
    for s in range(steps):
        q, tk, tv = rnd(rng, U, d), rnd(rng, U, d), rnd(rng, U, d)
        res = cache.decode(dev(q)[:, None, :].contiguous(), dev(tk), dev(tv), weights=weights,
                           scale_logits=scale)
        out, w = res if weights else (res, None)
        out = out.cpu().numpy()
        w = w.cpu().numpy() if weights else None
        for u in range(U):
            ro, rw = refs[u].decode(q[u], tk[u], tv[u], scale_logits=scale, weights=True)
            worst_out = max(worst_out, rel_l2(out[u, 0], ro))
            if weights:
                worst_w = max(worst_w, float(np.max(np.abs(w[u, 0] - rw))))
    return worst_out, worst_w


@pytest.mark.parametrize("cfg", [(2, 4, 8, 8), (2, 8, 16, 32), (4, 8, 16, 32), (8, 4, 8, 4),
                                 (2, 32, 128, 128), (1, 16, 32, 64), (2, 2, 2, 2)])
@pytest.mark.parametrize("l0", [1, 5, 17, 40])
def test_decode_generic_vs_reference(cuda, cfg, l0):
    e_out, e_w = run_decode(cfg, U=2, l0=l0 * cfg[2] // 8 + 1, steps=6, path="generic",
                            seed=l0 * 31 + cfg[0])
    assert e_out <= 1e-6, e_out
    assert e_w <= 1e-6, e_w


ROUTES = {"body": ("0", "0"), "small": ("1", "0"), "small_fused": ("1", "1")}


@pytest.mark.parametrize("route", sorted(ROUTES))
@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("l0", [1, 31, 127, 128, 129, 255, 256, 257, 383, 600, 1153])
def test_decode_fast_vs_reference(cuda, bits, l0, route, monkeypatch):
    # body: body + residual kernels; small: every token through 64-token items
    # (few-unit route); small_fused: the same in one cooperative launch that
    # also appends and merges
    monkeypatch.setenv("KIVI_SMALL_ITEMS", ROUTES[route][0])
    monkeypatch.setenv("KIVI_SMALL_FUSED", ROUTES[route][1])
    cfg = (bits, 32, 128, 128)
    e_out, e_w = run_decode(cfg, U=3, l0=l0, steps=4, path="fast", seed=l0 + bits)
    assert e_out <= 1e-5, e_out
    assert e_w <= 1e-5, e_w


@pytest.mark.parametrize("sub", ["384", "512", "-1"])
@pytest.mark.parametrize("vimma", ["1", "0"])
@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("l0", [1100, 1535, 2049])
def test_body_item_sizes(cuda, bits, l0, vimma, sub, monkeypatch):
    """The body kernel's 384- and 512-token items (KIVI_BODY_SUB fixes the
    size; -1, the default, takes the size covering the most tokens), with
    weights."""
    monkeypatch.setenv("KIVI_BODY_SUB", sub)
    monkeypatch.setenv("KIVI_SMALL_ITEMS", "0")
    monkeypatch.setenv("KIVI_VIMMA", vimma)
    e_out, e_w = run_decode((bits, 32, 128, 128), U=3, l0=l0, steps=4, path="fast",
                            seed=l0 + bits + 7)
    assert e_out <= 1e-5, e_out
    assert e_w <= 1e-5, e_w


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("qpk", [1, 4])
def test_combine_modes(cuda, mode, qpk, monkeypatch):
    """Every K5 merge mode (serial per thread, block-parallel, one warp per row)
    against the reference, MHA and GQA, with weights (the merge's (M, L) stats)."""
    monkeypatch.setenv("KIVI_COMBINE_PARALLEL", mode)
    monkeypatch.setenv("KIVI_SMALL_ITEMS", "0")
    ck = checker()
    rng = np.random.default_rng(17 + qpk + int(mode))
    U, l0, d = 5, 1300, 128
    K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
    cache = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    cache.prefill(dev(K), dev(V))
    refs = [[ck.unit(2, 32, 128, d) for _ in range(qpk)] for _ in range(U)]
    for u in range(U):
        for r in refs[u]:
            r.prefill(K[u], V[u])
    for step in range(3):
        q = rnd(rng, U, qpk, d)
        tk, tv = rnd(rng, U, d), rnd(rng, U, d)
        use_w = step == 2
        res = cache.decode(dev(q), dev(tk), dev(tv), q_per_kv=qpk, weights=use_w)
        out, w = res if use_w else (res, None)
        out = out.cpu().numpy()
        for u in range(U):
            for h in range(qpk):
                ro, rw = refs[u][h].decode(q[u, h], tk[u], tv[u], weights=True)
                assert rel_l2(out[u, h], ro) <= 1e-5, f"mode {mode} step {step} unit {u} head {h}"
                if use_w:
                    assert float(np.max(np.abs(w[u, h].cpu().numpy() - rw))) <= 1e-5
    cache.close()


@pytest.mark.parametrize("small", ["0", "1"])
@pytest.mark.parametrize("qpk", [1, 4])
def test_layers_interleaved_on_one_stream(cuda, small, qpk, monkeypatch):
    """A decode step over several layers: the caches' decodes are enqueued back to
    back on one stream with no host sync (the programmatic launches of one layer
    follow the previous layer's combine), each layer checked against its own
    reference units."""
    monkeypatch.setenv("KIVI_SMALL_ITEMS", small)
    ck = checker()
    rng = np.random.default_rng(41 + qpk)
    bits, G, R, d = 2, 32, 128, 128
    U, L, l0, steps = 3, 3, 700, 3
    caches, refs = [], []
    for _ in range(L):
        K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
        c = kb.KVCache(kb.CacheConfig(bits, G, R, d), U)
        c.set_attend_path("fast")
        c.prefill(dev(K), dev(V))
        caches.append(c)
        rs = [ck.unit(bits, G, R, d) for _ in range(U * qpk)]
        for u in range(U):
            for h in range(qpk):
                rs[u * qpk + h].prefill(K[u], V[u])
        refs.append(rs)
    worst = 0.0
    for _ in range(steps):
        ins = [(rnd(rng, U, qpk, d), rnd(rng, U, d), rnd(rng, U, d)) for _ in range(L)]
        outs = [c.decode(dev(q), dev(tk), dev(tv), q_per_kv=qpk)
                for c, (q, tk, tv) in zip(caches, ins)]
        for li in range(L):
            q, tk, tv = ins[li]
            o = outs[li].cpu().numpy()
            for u in range(U):
                for h in range(qpk):
                    ro = refs[li][u * qpk + h].decode(q[u, h], tk[u], tv[u], scale_logits=True)
                    worst = max(worst, rel_l2(o[u, h], ro))
    assert worst <= 5e-5 if qpk > 1 else worst <= 1e-5, worst


@pytest.mark.parametrize("route", [("0", "1", "0"), ("0", "0", "0"), ("1", "0", "0"),
                                   ("1", "0", "1")])
@pytest.mark.parametrize("bits", [2, 4])
def test_decode_fast_across_flush_and_long_context(cuda, bits, route, monkeypatch):
    # (small items, fused append, single-launch small route) across 130 value
    # pops and a key flush: the fused routes append inside the attend launch
    monkeypatch.setenv("KIVI_SMALL_ITEMS", route[0])
    monkeypatch.setenv("KIVI_FUSED_APPEND", route[1])
    monkeypatch.setenv("KIVI_SMALL_FUSED", route[2])
    cfg = (bits, 32, 128, 128)
    # 130 steps cross a key flush and 130 value pops; ctx ~4k like config 1.
    e_out, _ = run_decode(cfg, U=2, l0=3968, steps=130, path="fast", seed=7, weights=False)
    assert e_out <= 1e-5, e_out


def test_fast_equals_generic_closely(cuda):
    rng = np.random.default_rng(3)
    U, d, l0 = 8, 128, 2000
    K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
    a = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    a.prefill(dev(K), dev(V))
    b = a.clone()
    a.set_attend_path("fast")
    b.set_attend_path("generic")
    q = dev(rnd(rng, U, 1, d))
    oa = a.attend(q).cpu().numpy()
    ob = b.attend(q).cpu().numpy()
    for u in range(U):
        assert rel_l2(oa[u], ob[u]) <= 1e-5


def test_profile_stride_times_every_kth_attend(cuda):
    """kivi_profile_enable(k): events around every k-th attend launch only
    (bench.py samples so the events' host cost stays off latency-bound steps)."""
    rng = np.random.default_rng(5)
    U, d, l0 = 4, 128, 300
    K = rnd(rng, U, l0, d)
    c = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    c.prefill(dev(K), dev(K))
    q = dev(rnd(rng, U, 1, d))
    c.profile_enable(3)
    for _ in range(7):
        c.attend(q)
    ms, n, tot = c.profile_read()
    assert n == 3 and ms > 0 and tot >= 7  # launches 0, 3, 6 timed
    c.profile_enable(1)
    c.attend(q)
    c.attend(q)
    assert c.profile_read()[1] == 2
    c.profile_enable(False)
    c.attend(q)
    assert c.profile_read()[1] == 0
    with pytest.raises(kb.UsageError):
        c.profile_enable(-1)


def run_gqa(cfg, U, qpk, l0, steps, path, seed, weights=False, kscale=1.0, vscale=1.0,
            qscale=1.0, outliers=()):
    """GQA: one append per unit, q_per_kv query heads; the reference emulates
    each head with its own state copy.  kscale/vscale/qscale and
    key outlier channels (x50, analysis.hpp:59-61) move the operand ranges the
    tensor-core path rescales per job."""
    ck = checker()
    rng = np.random.default_rng(seed)
    bits, G, R, d = cfg
    K, V = rnd(rng, U, l0, d, scale=kscale), rnd(rng, U, l0, d, scale=vscale)
    for c in outliers:
        K[:, :, c] *= 50.0
    cache = kb.KVCache(kb.CacheConfig(*cfg), U)
    cache.set_attend_path(path)
    cache.prefill(dev(K), dev(V))
    refs = [[ck.unit(*cfg) for _ in range(qpk)] for _ in range(U)]
    for u in range(U):
        for h in range(qpk):
            refs[u][h].prefill(K[u], V[u])
    worst, worst_w = 0.0, 0.0
    for _ in range(steps):
        q = rnd(rng, U, qpk, d, scale=qscale)
        tk, tv = rnd(rng, U, d, scale=kscale), rnd(rng, U, d, scale=vscale)
        for c in outliers:
            tk[:, c] *= 50.0
        res = cache.decode(dev(q), dev(tk), dev(tv), q_per_kv=qpk, weights=weights)
        out, w = res if weights else (res, None)
        out = out.cpu().numpy()
        for u in range(U):
            for h in range(qpk):
                ro, rw = refs[u][h].decode(q[u, h], tk[u], tv[u], weights=True)
                worst = max(worst, rel_l2(out[u, h], ro))
                if weights:
                    worst_w = max(worst_w, float(np.max(np.abs(w[u, h].cpu().numpy() - rw))))
    return worst, worst_w


def test_gqa_generic_matches_per_head_reference(cuda):
    e, _ = run_gqa((2, 32, 128, 128), U=2, qpk=4, l0=300, steps=2, path="generic", seed=9)
    assert e <= 1e-6, e


@pytest.mark.parametrize("qpk", [2, 4])
@pytest.mark.parametrize("l0", [1, 100, 255, 256, 300, 777])
def test_gqa_fast_vs_reference(cuda, qpk, l0):
    e, ew = run_gqa((2, 32, 128, 128), U=3, qpk=qpk, l0=l0, steps=3, path="fast", seed=l0 + qpk,
                    weights=True)
    assert e <= 1e-5, e
    assert ew <= 1e-5, ew


@pytest.mark.parametrize("small", ["0", "1"])
@pytest.mark.parametrize("bits,qpk", [(4, 2), (4, 4), (2, 3), (2, 6), (2, 8), (4, 8)])
def test_gqa_heads_route(cuda, bits, qpk, small, monkeypatch):
    """GQA shapes outside the tensor-core kernel (4-bit, or q_per_kv not in
    {2, 4}) take one MHA fast attend per query head over the shared cache
    (attend_heads_mha) -- with weights, through the body and few-unit routes,
    across a key flush -- instead of the generic kernel."""
    monkeypatch.setenv("KIVI_SMALL_ITEMS", small)
    l0 = 1150 if small == "0" else 380
    e, ew = run_gqa((bits, 32, 128, 128), U=3, qpk=qpk, l0=l0, steps=3, path="fast",
                    seed=bits * 10 + qpk, weights=True)
    assert e <= 1e-5, e
    assert ew <= 1e-5, ew


@pytest.mark.parametrize("qpk", [2, 4])
def test_gqa_384_token_items(cuda, qpk, monkeypatch):
    """The tensor-core GQA body with 384-token items (KIVI_GQA_ITEM=384, off by
    default: its longer truncating accumulation costs accuracy on outlier
    channels), on ordinary operands across a partial last item, with weights."""
    monkeypatch.setenv("KIVI_GQA_ITEM", "384")
    for l0 in (1100, 1500):
        e, ew = run_gqa((2, 32, 128, 128), U=3, qpk=qpk, l0=l0, steps=2, path="fast",
                        seed=l0 + qpk, weights=True)
        assert e <= 1e-5, e
        assert ew <= 1e-5, ew


# (kscale, vscale, qscale, key outlier channels, tolerance).  The last case
# has log2-domain logits of magnitude ~500: one fp32 ulp there is 3e-5, so
# even the reference's own float cast of its double logits (attention.cpp:59-62)
# moves the softmax by that much; the bar scales with the logit magnitude.
@pytest.mark.parametrize("qpk", [2, 4])
@pytest.mark.parametrize("scales", [(1e-3, 1e-3, 1.0, (), 1e-5), (30.0, 200.0, 3.0, (), 1e-5),
                                    (1.0, 1.0, 1.0, (1, 17, 40), 1e-5),
                                    (4.0, 0.01, 20.0, (5,), 5e-5)])
def test_gqa_fast_operand_ranges(cuda, qpk, scales):
    # the tensor-core body path scales its fp16 operands by 2^E per job and
    # must keep fp32-class accuracy on 50x outlier key channels
    ks, vs, qs, outl, tol = scales
    e, ew = run_gqa((2, 32, 128, 128), U=3, qpk=qpk, l0=1100, steps=2, path="fast",
                    seed=int(ks * 10 + vs) + qpk, weights=True, kscale=ks, vscale=vs, qscale=qs,
                    outliers=outl)
    assert e <= tol, e
    assert ew <= tol, ew


def test_gqa_fast_across_flush(cuda):
    e, _ = run_gqa((2, 32, 128, 128), U=2, qpk=4, l0=2000, steps=130, path="fast", seed=77)
    assert e <= 1e-5, e


def test_single_token_exact(cuda):
    # reference test_attention.cpp:52-63
    rng = np.random.default_rng(32)
    cache = kb.KVCache(kb.CacheConfig(2, 4, 8, 4), 1)
    q, tk, tv = rnd(rng, 1, 1, 4), rnd(rng, 1, 4), rnd(rng, 1, 4)
    out, w = cache.decode(dev(q), dev(tk), dev(tv), weights=True)
    assert out.cpu().numpy().reshape(-1).tobytes() == tv.reshape(-1).tobytes()
    assert w.cpu().numpy().reshape(-1).tolist() == [1.0]


def test_passthrough_bit_exact(cuda):
    # reference test_attention.cpp:84-103: R >= l keeps everything fp32, and the
    # decode equals reference_attention over the concatenated rows bitwise.
    rng = np.random.default_rng(34)
    for trial in range(10):
        for d in (32, 64):
            l = int(rng.integers(1, 301))
            K, V = rnd(rng, 1, l, d), rnd(rng, 1, l, d)
            cache = kb.KVCache(kb.CacheConfig(2, 32, 512, d), 1)
            cache.prefill(dev(K), dev(V))
            q, tk, tv = rnd(rng, 1, 1, d), rnd(rng, 1, d), rnd(rng, 1, d)
            out = cache.decode(dev(q), dev(tk), dev(tv)).cpu().numpy().reshape(-1)
            Kc = np.concatenate([K[0], tk], 0)
            Vc = np.concatenate([V[0], tv], 0)
            ref = kb.reference_attention(dev(q[0]), dev(Kc), dev(Vc)).cpu().numpy().reshape(-1)
            assert out.tobytes() == ref.tobytes()


def test_reference_attention_vs_reference(cuda):
    ck = checker()
    rng = np.random.default_rng(31)
    for l, d, nq in ((1, 4, 1), (5, 3, 2), (300, 64, 3)):
        q, K, V = rnd(rng, nq, d), rnd(rng, l, d), rnd(rng, l, d)
        got = kb.reference_attention(dev(q), dev(K), dev(V)).cpu().numpy()
        want = ck.reference_attention(q, K, V)
        assert rel_l2(got, want) <= 1e-6


def test_host_buffers_path_equals_device_path(cuda):
    rng = np.random.default_rng(77)
    U, d = 16, 128
    K, V = rnd(rng, U, 700, d), rnd(rng, U, 700, d)
    a = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    a.prefill_host(K, V)
    b = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    b.prefill(dev(K), dev(V))
    for _ in range(3):
        q, tk, tv = rnd(rng, U, 1, d), rnd(rng, U, d), rnd(rng, U, d)
        out_h = np.zeros((U, 1, d), np.float32)
        a.decode_host(q, tk, tv, out_h)
        a.host_join()
        torch.cuda.current_stream().synchronize()
        out_d = b.decode(dev(q), dev(tk), dev(tv)).cpu().numpy()
        assert out_h.tobytes() == out_d.tobytes()


def test_errors(cuda):
    with pytest.raises(kb.ConfigError):
        kb.KVCache(kb.CacheConfig(2, 32, 100, 64), 1)   # R % G != 0
    with pytest.raises(kb.ConfigError):
        kb.KVCache(kb.CacheConfig(2, 32, 128, 50), 1)   # d % G != 0
    with pytest.raises(kb.ConfigError):
        kb.KVCache(kb.CacheConfig(3, 2, 4, 2), 1)       # not packable
    c = kb.KVCache(kb.CacheConfig(2, 2, 4, 2), 1)
    with pytest.raises(kb.UsageError):
        c.prefill(torch.zeros((1, 0, 2), device="cuda"), torch.zeros((1, 0, 2), device="cuda"))
    with pytest.raises(kb.ShapeError):
        c.append(torch.zeros((1, 3), device="cuda"), torch.zeros((1, 2), device="cuda"))


def test_capacity_grows_on_append(cuda):
    rng = np.random.default_rng(5)
    c = kb.KVCache(kb.CacheConfig(2, 4, 8, 8), 2, capacity_tokens=8)
    ck = checker()
    refs = [ck.unit(2, 4, 8, 8) for _ in range(2)]
    for t in range(50):
        tk, tv = rnd(rng, 2, 8), rnd(rng, 2, 8)
        c.append(dev(tk), dev(tv))
        for u in range(2):
            refs[u].append(tk[u], tv[u])
    for u in range(2):
        assert_state_equal(c.export_unit(u), refs[u].export())


def test_import_export_roundtrip(cuda):
    ck = checker()
    rng = np.random.default_rng(8)
    cfg = (2, 8, 16, 32)
    r = ck.unit(*cfg)
    r.prefill(rnd(rng, 77, 32), rnd(rng, 77, 32))
    st = r.export()
    cnt = r.counters()
    c = kb.KVCache(kb.CacheConfig(*cfg), 1)
    c.import_unit(0, int(cnt["total"]), int(cnt["key_capacity"]), int(cnt["value_capacity"]), st)
    assert_state_equal(c.export_unit(0), st)
    q, tk, tv = rnd(rng, 32), rnd(rng, 32), rnd(rng, 32)
    out = c.decode(dev(q)[None, None], dev(tk)[None], dev(tv)[None]).cpu().numpy().reshape(-1)
    assert rel_l2(out, r.decode(q, tk, tv)) <= 1e-6


# ---- workload driver (reference run_decode_benchmark, workload.cpp:145-271) ----

def test_run_decode_benchmark_matches_reference_tiny(cuda):
    """The reference's own synthetic data (tests/golden/workload_tiny.npz): same
    checksum of every decode output (tolerance: fp32 GEMM order), identical peak
    cache bytes counted from live states, both modes."""
    import json
    from paper_2402_02750_b200 import workload as wl
    here = os.path.join(os.path.dirname(__file__), "golden")
    gold = json.load(open(os.path.join(here, "workload_golden.json")))["tiny_run"]
    data = np.load(os.path.join(here, "workload_tiny.npz"))
    sp = wl.WorkloadSpec(*gold["spec"])
    bits, G, R = gold["cfg"]
    for mode in ("kivi", "fp"):
        rep = wl.run_decode_benchmark(sp, kb.CacheConfig(bits, G, R, sp.head_dim), mode=mode,
                                      data=(data["weights"], data["prompts"], data["tokens"]))
        want = gold["reference"][mode]
        assert rep.peak_cache_bytes == want["peak_cache_bytes"], mode
        assert abs(rep.output_checksum - want["output_checksum"]) <= 1e-5 * rep.output_abs_sum, \
            (mode, rep.output_checksum, want["output_checksum"], rep.output_abs_sum)
        assert rep.decode_steps == sp.gen_len and rep.tokens_per_sec > 0


def test_run_decode_benchmark_fast_path_vs_reference(cuda):
    """d = 128, G = 32, R = 128 (the fast kernels), data from the reference."""
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=3, prompt_len=700, gen_len=5, layers=2, kv_heads=2, head_dim=128)
    ref = Ref()
    data = ref.workload_data(sp, 3)
    want = ref.run_decode_benchmark(sp, 3, 0, 2, 32, 128)
    rep = wl.run_decode_benchmark(sp, kb.CacheConfig(2, 32, 128, 128), data=data,
                                  fused_projection=False)
    assert rep.peak_cache_bytes == want["peak_cache_bytes"]
    assert abs(rep.output_checksum - want["output_checksum"]) <= 1e-5 * rep.output_abs_sum
    # the fused tensor-core projection + append: same bar
    fused = wl.run_decode_benchmark(sp, kb.CacheConfig(2, 32, 128, 128), data=data)
    assert fused.peak_cache_bytes == want["peak_cache_bytes"]
    assert abs(fused.output_checksum - want["output_checksum"]) <= 1e-5 * fused.output_abs_sum


def test_run_decode_benchmark_fused_projection_no_library_gemm(cuda, monkeypatch):
    """At d = 128 the driver's q/k/v projections run on the tcgen05 projection
    kernel fused with the append (kivi_proj_append / kivi_proj_gemm): no
    torch.matmul anywhere on the prefill or decode path."""
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=2, prompt_len=300, gen_len=6, layers=2, kv_heads=2, head_dim=128)
    cfg = kb.CacheConfig(2, 32, 128, 128)
    want = wl.run_decode_benchmark(sp, cfg, seed=4, fused_projection=False)

    def no_gemm(*a, **k):
        raise AssertionError("library GEMM on the fused decode path")
    monkeypatch.setattr(torch, "matmul", no_gemm)
    rep = wl.run_decode_benchmark(sp, cfg, seed=4, fused_projection=True)
    # same checksum as the cuBLAS-projected run, to the reference driver's own
    # tolerance (fp32 GEMMs in another order, test_run_decode_benchmark_*)
    assert rep.decode_steps == sp.gen_len and rep.peak_cache_bytes == want.peak_cache_bytes
    assert abs(rep.output_checksum - want.output_checksum) <= 1e-5 * rep.output_abs_sum, \
        (rep.output_checksum, want.output_checksum, rep.output_abs_sum)


def test_native_driver_vs_reference(cuda):
    """The C++ driver (kivi_run_decode_benchmark, libkivi_driver.so) fed the
    reference's own draws reproduces its checksum and peak bytes."""
    if not Ref.available():
        pytest.skip("oracle/_ref not built")
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=3, prompt_len=700, gen_len=5, layers=2, kv_heads=2, head_dim=128)
    ref = Ref()
    data = ref.workload_data(sp, 3)
    want = ref.run_decode_benchmark(sp, 3, 0, 2, 32, 128)
    rep = wl.run_decode_benchmark_native(sp, kb.CacheConfig(2, 32, 128, 128), data=data)
    assert rep.peak_cache_bytes == want["peak_cache_bytes"]
    assert abs(rep.output_checksum - want["output_checksum"]) <= 1e-5 * rep.output_abs_sum
    assert rep.decode_steps == sp.gen_len and rep.tokens_per_sec > 0 and rep.p50_ms > 0


def test_native_driver_threads_and_budget(cuda):
    """One host thread per device entry (here two threads sharing cuda:0, the
    batch split in two blocks) gives the single-thread result; peak bytes
    equal estimate_memory (counted == estimated) and a budget one byte short
    raises BudgetError (workload.cpp:175-192)."""
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=5, prompt_len=260, gen_len=9, layers=2, kv_heads=2, head_dim=128)
    cfg = kb.CacheConfig(2, 32, 128, 128)
    one = wl.run_decode_benchmark_native(sp, cfg, seed=11, devices=(0,))
    two = wl.run_decode_benchmark_native(sp, cfg, seed=11, devices=(0, 0))
    assert one.peak_cache_bytes == two.peak_cache_bytes == wl.estimate_memory(sp, cfg).kivi_bytes
    assert abs(one.output_checksum - two.output_checksum) <= 1e-5 * one.output_abs_sum
    assert abs(one.output_abs_sum - two.output_abs_sum) <= 1e-5 * one.output_abs_sum
    est = wl.estimate_memory(sp, cfg).kivi_bytes
    wl.run_decode_benchmark_native(sp, cfg, seed=11, budget_bytes=est)
    with pytest.raises(kb.BudgetError):
        wl.run_decode_benchmark_native(sp, cfg, seed=11, budget_bytes=est - 1)


def test_run_decode_benchmark_budget(cuda):
    from paper_2402_02750_b200 import workload as wl
    sp = wl.WorkloadSpec(batch=2, prompt_len=100, gen_len=40, layers=1, kv_heads=2, head_dim=128)
    cfg = kb.CacheConfig(2, 32, 128, 128)
    est = wl.estimate_memory(sp, cfg).kivi_bytes
    rep = wl.run_decode_benchmark(sp, cfg, seed=1, budget_bytes=est)
    assert rep.peak_cache_bytes == est  # counted == estimated (reference acceptance c5)
    with pytest.raises(kb.BudgetError):
        wl.run_decode_benchmark(sp, cfg, seed=1, budget_bytes=est - 1)


def test_export_cache_unit_kvqd(cuda, tmp_path):
    """A device cache unit dumped as KVQD equals the reference's materialisation
    of the same state (read back by the reference's own read_dump when built)."""
    from paper_2402_02750_b200.dump_io import export_cache_unit, read_dump
    ck = checker()
    rng = np.random.default_rng(21)
    U, d, l0 = 3, 128, 333
    K, V = rnd(rng, U, l0, d), rnd(rng, U, l0, d)
    cache = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    cache.prefill(dev(K), dev(V))
    kp, vp = str(tmp_path / "k.kvqd"), str(tmp_path / "v.kvqd")
    export_cache_unit(cache, 1, kp, vp)
    r = ck.unit(2, 32, 128, d)
    r.prefill(K[1], V[1])
    mk, mv = r.materialize()
    (gk,), (gv,) = read_dump(kp), read_dump(vp)
    assert gk.tobytes() == np.asarray(mk, np.float32).tobytes()
    assert gv.tobytes() == np.asarray(mv, np.float32).tobytes()
    if Ref.available():
        back, err = Ref().read_dump(kp)
        assert err is None and back[0].tobytes() == gk.tobytes()


@pytest.mark.parametrize("graph", ["0", "1"])
@pytest.mark.parametrize("qpk,U,l0", [(1, 3, 700), (1, 64, 2300), (1, 80, 2300), (4, 4, 900)])
def test_decode_layers_equals_per_layer(cuda, graph, qpk, U, l0, monkeypatch):
    """kivi_decode_layers / kivi_decode_layers_host (one call per model step,
    optionally replayed as a CUDA graph) give bit-identical outputs and states
    to per-layer kivi_decode calls, across a key flush."""
    monkeypatch.setenv("KIVI_SMALL_ITEMS", "1")
    monkeypatch.setenv("KIVI_STEP_GRAPH", graph)
    rng = np.random.default_rng(60 + U + qpk)
    L, d = 3, 128
    cfg = kb.CacheConfig(2, 32, 128, d)
    mk = []
    for _ in range(3):
        cs = []
        for ly in range(L):
            K = rnd(np.random.default_rng(ly), U, l0, d)
            c = kb.KVCache(cfg, U)
            c.prefill(dev(K), dev(K * 0.5))
            cs.append(c)
        mk.append(cs)
    ref, devs, host = mk
    sd, sh = kb.LayerStack(devs), kb.LayerStack(host)
    stream = torch.cuda.Stream()
    hq = torch.empty((L, U, qpk, d), pin_memory=True)
    hk = torch.empty((L, U, d), pin_memory=True)
    hv = torch.empty((L, U, d), pin_memory=True)
    ho = torch.empty((L, U, qpk, d), pin_memory=True)
    for step in range(l0 % 128 and 130 - l0 % 128 or 3):
        q, tk, tv = rnd(rng, L, U, qpk, d), rnd(rng, L, U, d), rnd(rng, L, U, d)
        want = np.stack([ref[ly].decode(dev(q[ly]), dev(tk[ly]), dev(tv[ly]), q_per_kv=qpk)
                         .cpu().numpy() for ly in range(L)])
        od = torch.empty((L, U, qpk, d), device="cuda")
        sd.decode(dev(q), dev(tk), dev(tv), od, q_per_kv=qpk)
        hq.copy_(torch.from_numpy(q))
        hk.copy_(torch.from_numpy(tk))
        hv.copy_(torch.from_numpy(tv))
        with torch.cuda.stream(stream):
            sh.decode_host(hq, hk, hv, ho, q_per_kv=qpk, stream=stream)
        assert od.cpu().numpy().tobytes() == want.tobytes(), step
        assert ho.numpy().tobytes() == want.tobytes(), step
    torch.cuda.synchronize()
    if graph == "1":
        stats = kb.step_graph_stats()
        assert stats["capture_failed"] == 0 and stats["replayed"] > 0, stats
    for ly in range(L):
        for u in (0, U - 1):
            a, b, c = ref[ly].export_unit(u), devs[ly].export_unit(u), host[ly].export_unit(u)
            for key in a:
                assert a[key].tobytes() == b[key].tobytes() == c[key].tobytes(), (ly, u, key)


@pytest.mark.parametrize("on_stream", [False, True])
@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("qpk,U,l0", [(1, 32, 4000), (4, 8, 900)])
def test_decode_layers_host_single_layer_zero_copy(cuda, pinned, qpk, U, l0, on_stream,
                                                   monkeypatch):
    """One layer through kivi_decode_layers_host: with pinned buffers the
    append reads the key/value rows and the merge writes the outputs across
    PCIe (zero-copy); pageable buffers take the copy path.  Both equal
    kivi_decode on device rows bit for bit, across a key flush.  On a stream
    of its own the step is replayed as a CUDA graph by default (single-layer
    steps, KIVI_STEP_GRAPH unset)."""
    monkeypatch.delenv("KIVI_STEP_GRAPH", raising=False)
    stream = torch.cuda.Stream() if on_stream else None
    replayed0 = kb.step_graph_stats()["replayed"]
    rng = np.random.default_rng(90 + U + qpk)
    d = 128
    cfg = kb.CacheConfig(2, 32, 128, d)
    K = rnd(np.random.default_rng(7), U, l0, d)
    ref, host = kb.KVCache(cfg, U), kb.KVCache(cfg, U)
    for c in (ref, host):
        c.prefill(dev(K), dev(K * 0.5))
    sh = kb.LayerStack([host])
    mk = (lambda shape: torch.empty(shape, pin_memory=True)) if pinned else torch.empty
    hq, hk, hv, ho = mk((1, U, qpk, d)), mk((1, U, d)), mk((1, U, d)), mk((1, U, qpk, d))
    for step in range(130 - l0 % 128):
        q, tk, tv = rnd(rng, 1, U, qpk, d), rnd(rng, 1, U, d), rnd(rng, 1, U, d)
        want = ref.decode(dev(q[0]), dev(tk[0]), dev(tv[0]), q_per_kv=qpk).cpu().numpy()
        hq.copy_(torch.from_numpy(q))
        hk.copy_(torch.from_numpy(tk))
        hv.copy_(torch.from_numpy(tv))
        if stream is None:
            sh.decode_host(hq, hk, hv, ho, q_per_kv=qpk)
        else:
            with torch.cuda.stream(stream):
                sh.decode_host(hq, hk, hv, ho, q_per_kv=qpk, stream=stream)
        assert ho.numpy()[0].tobytes() == want.tobytes(), step
    torch.cuda.synchronize()
    stats = kb.step_graph_stats()
    assert stats["capture_failed"] == 0
    if on_stream:
        assert stats["replayed"] > replayed0, stats
    for u in (0, U - 1):
        a, b = ref.export_unit(u), host.export_unit(u)
        for key in a:
            assert a[key].tobytes() == b[key].tobytes(), (u, key)


@pytest.mark.parametrize("vimma", ["1", "0"])
@pytest.mark.parametrize("growth", ["rising", "falling", "spiky"])
def test_body_value_spans_change_between_jobs(cuda, vimma, growth, monkeypatch):
    """The body's value jobs on the integer tensor cores keep a fixed-point
    scale per channel group and item; a later job with larger spans moves the
    integer sums to fp32 (regression: shifting the digit columns one by one
    lost up to 2^24 units).  Value magnitudes that rise, fall or spike along
    the sequence force every case; outputs vs the reference, 1e-5."""
    monkeypatch.setenv("KIVI_VIMMA", vimma)
    ck = checker()
    rng = np.random.default_rng({"rising": 1, "falling": 2, "spiky": 3}[growth])
    U, d, l0 = 40, 128, 1500
    t = np.arange(l0, dtype=np.float32)[None, :, None]
    if growth == "rising":
        mag = 2.0 ** (t / 300.0)
    elif growth == "falling":
        mag = 2.0 ** (-(t / 300.0))
    else:
        mag = np.where((t.astype(np.int64) // 64) % 3 == 1, 8.0, 1.0).astype(np.float32)
    K = rnd(rng, U, l0, d)
    V = (rnd(rng, U, l0, d) * mag).astype(np.float32)
    cache = kb.KVCache(kb.CacheConfig(2, 32, 128, d), U)
    cache.prefill(dev(K), dev(V))
    units = (0, 7, 19, U - 1)
    refs = {u: ck.unit(2, 32, 128, d) for u in units}
    for u in units:
        refs[u].prefill(K[u], V[u])
    for step in range(3):
        q, tk, tv = rnd(rng, U, 1, d), rnd(rng, U, d), rnd(rng, U, d)
        out = cache.decode(dev(q), dev(tk), dev(tv)).cpu().numpy()
        for u in units:
            want = refs[u].decode(q[u, 0], tk[u], tv[u])
            err = rel_l2(out[u, 0], want)
            assert err <= 1e-5, (growth, step, u, err)
    cache.close()
