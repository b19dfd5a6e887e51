"""CPU: pin the plain-C restatement (oracle/liboracle.so) to the reference.

* golden vectors produced by the reference itself (tests/golden/make_golden.py
  runs oracle/_ref, the reference compiled from its own sources);
* the known-answer tests the reference's own unit tests hold
  (reference proj/tests/test_quantize.cpp:42-108, test_kv_cache.cpp:30-98,
  test_attention.cpp:52-63);
* when oracle/_ref is present: the reference's own unit + acceptance suites
  (compiled verbatim against this repo's Eigen/doctest subsets) pass.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracles import ROOT, Port, Ref, rel_l2

GOLD = os.path.join(ROOT, "tests", "golden", "kivi_golden.npz")
MANIFEST = os.path.join(ROOT, "tests", "golden", "kivi_golden.json")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def manifest():
    with open(MANIFEST) as f:
        return json.load(f)


def test_counter_rng_matches_numpy():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import uniform
    assert uniform(257, 11, 3).tobytes() == Port().uniform(257, 11, 3).tobytes()


def test_quantize_group_goldens(gold, manifest):
    p = Port()
    for i in range(manifest["groups"]):
        bits = int(gold[f"g{i}_bits"][0])
        codes, z, s = p.quantize_group(gold[f"g{i}_in"], bits)
        assert codes.tobytes() == gold[f"g{i}_codes"].tobytes(), i
        assert np.array([z, s]).tobytes() == gold[f"g{i}_zs"].tobytes(), i


def test_pack_goldens(gold):
    p = Port()
    for bits in (1, 2, 4, 8):
        assert p.pack_codes(gold[f"pack{bits}_codes"], bits).tobytes() == \
            gold[f"pack{bits}_bytes"].tobytes()


def test_matrix_goldens(gold, manifest):
    p = Port()
    for i, (rows, cols, bits, G, pc) in enumerate(manifest["matrices"]):
        pk, z, s = p.quantize_matrix(gold[f"m{i}_in"], bits, G, pc)
        assert pk.tobytes() == gold[f"m{i}_packed"].tobytes()
        assert z.tobytes() == gold[f"m{i}_z"].tobytes()
        assert s.tobytes() == gold[f"m{i}_s"].tobytes()


def test_trace_goldens(gold, manifest):
    """Streaming cache + decode: the port is arithmetic-identical to the
    reference (same operation order, no FMA contraction): bit-exact."""
    p = Port()
    for ti, (bits, G, R, d, l0, steps, _seed) in enumerate(manifest["traces"]):
        pre = f"t{ti}_"
        K, V, Q = gold[pre + "K"], gold[pre + "V"], gold[pre + "Q"]
        u = p.unit(bits, G, R, d)
        u.prefill(K[:l0], V[:l0])
        for s in range(steps):
            o, w = u.decode(Q[s], K[l0 + s], V[l0 + s], weights=True)
            assert o.tobytes() == gold[pre + "out"][s].tobytes(), (ti, s)
        assert w.tobytes() == gold[pre + "w_last"].tobytes()
        st = u.export()
        for k in st:
            assert st[k].tobytes() == gold[pre + k].tobytes(), (ti, k)
        c = u.counters()
        got = [c[k] for k in ("key_grouped", "key_residual", "total", "key_capacity",
                              "value_grouped", "value_residual", "value_capacity",
                              "key_memory", "value_memory")]
        assert np.array(got, np.int64).tobytes() == gold[pre + "counters"].tobytes()
        km, vm = u.materialize()
        assert km.tobytes() == gold[pre + "mat_k"].tobytes()
        assert vm.tobytes() == gold[pre + "mat_v"].tobytes()


def test_reference_attention_golden(gold):
    got = Port().reference_attention(gold["ra_q"], gold["ra_K"], gold["ra_V"])
    assert got.tobytes() == gold["ra_out"].tobytes()


def test_reference_known_answers():
    """Hand-written expectations of reference test_quantize.cpp:42-108."""
    p = Port()
    codes, z, s = p.quantize_group([0, 1, 2, 3], 2)
    assert codes.tolist() == [0, 1, 2, 3] and z == 0.0 and s == 1.0
    codes, z, s = p.quantize_group([1, 1, 1], 2)
    assert codes.tolist() == [0, 0, 0] and z == 1.0 and s == 1.0
    codes, z, s = p.quantize_group([0.0, 0.1, 0.9, 1.0], 2)
    assert codes.tolist() == [0, 0, 3, 3] and z == 0.0 and abs(s - 1 / 3) < 1e-15
    assert p.pack_codes([0, 1, 2, 3], 2).tolist() == [0xE4]
    assert p.pack_codes([3], 2).tolist() == [0x03]
    assert p.pack_codes([0xA, 0xB], 4).tolist() == [0xBA]
    from oracles import CheckerError
    with pytest.raises(CheckerError):
        p.quantize_group([], 2)
    with pytest.raises(CheckerError):
        p.pack_codes([4], 2)


def test_cache_split_arithmetic():
    """reference test_kv_cache.cpp:30-63 (prefill splits) and :65-98 (traces)."""
    p = Port()
    rng = np.random.default_rng(21)
    u = p.unit(2, 2, 4, 2)
    u.prefill(rng.uniform(-1, 1, (5, 2)), rng.uniform(-1, 1, (5, 2)))
    c = u.counters()
    assert (c["key_grouped"], c["key_residual"], c["value_grouped"], c["value_residual"]) == \
        (4, 1, 1, 4)
    u = p.unit(2, 2, 2, 2)
    u.prefill(rng.uniform(-1, 1, (2, 2)), rng.uniform(-1, 1, (2, 2)))
    u.append(rng.uniform(-1, 1, 2), rng.uniform(-1, 1, 2))
    assert u.counters()["key_residual"] == 1
    u.append(rng.uniform(-1, 1, 2), rng.uniform(-1, 1, 2))
    c = u.counters()
    assert (c["key_residual"], c["key_grouped"], c["value_residual"], c["value_grouped"]) == \
        (0, 4, 2, 2)


def test_single_token_exact():
    """reference test_attention.cpp:52-63."""
    rng = np.random.default_rng(32)
    u = Port().unit(2, 4, 8, 4)
    q, tk, tv = (rng.uniform(-1, 1, 4).astype(np.float32) for _ in range(3))
    o, w = u.decode(q, tk, tv, weights=True)
    assert o.tobytes() == tv.tobytes() and w.tolist() == [1.0]


def test_hybrid_vs_monolithic():
    """reference test_attention.cpp:65-82 on the port: rel-L2 <= 1e-5."""
    rng = np.random.default_rng(33)
    p = Port()
    for _ in range(10):
        l = int(rng.integers(1, 121))
        u = p.unit(2, 8, 16, 32)
        u.prefill(rng.uniform(-1, 1, (l, 32)), rng.uniform(-1, 1, (l, 32)))
        q, tk, tv = (rng.uniform(-1, 1, 32).astype(np.float32) for _ in range(3))
        o = u.decode(q, tk, tv)
        km, vm = u.materialize()
        ref = p.reference_attention(q[None], km, vm)[0]
        assert rel_l2(o, ref) <= 1e-5


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_port_equals_compiled_reference_random():
    p, r = Port(), Ref()
    rng = np.random.default_rng(99)
    for cfg in ((2, 32, 128, 128), (4, 4, 8, 8), (1, 2, 4, 6)):
        bits, G, R, d = cfg
        up, ur = p.unit(*cfg), r.unit(*cfg)
        l = int(rng.integers(1, 3 * R))
        K, V = rng.uniform(-2, 2, (l, d)), rng.uniform(-2, 2, (l, d))
        up.prefill(K, V)
        ur.prefill(K, V)
        for _ in range(R + 3):
            q, tk, tv = (rng.uniform(-1, 1, d).astype(np.float32) for _ in range(3))
            a, wa = up.decode(q, tk, tv, weights=True)
            b, wb = ur.decode(q, tk, tv, weights=True)
            assert a.tobytes() == b.tobytes() and wa.tobytes() == wb.tobytes()
        ea, eb = up.export(), ur.export()
        assert all(ea[k].tobytes() == eb[k].tobytes() for k in ea)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_unit")),
                    reason="oracle/_ref not built")
def test_reference_own_suites_pass_on_compiled_reference():
    """The reference's unit tests (test_{matrix,quantize,kv_cache,attention}.cpp)
    and acceptance criteria, compiled verbatim, pass against oracle/_ref —
    validating the Eigen/doctest subsets the checker is built with."""
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_unit")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_acceptance")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all criteria passed" in r.stdout
