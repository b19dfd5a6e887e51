"""GPU parity over randomly drawn shapes (seeded, reproducible): bits, group
size, residual length, head dim, units, query heads per kv head, prompt
length and decode steps drawn from what the reference accepts, so every
routing decision of the library (fast MHA body / few-unit route, tensor-core
GQA, per-head-group GQA passes, generic kernel) meets the reference on shapes
nobody picked by hand.  Bars: state bit-exact; outputs rel-L2 <= 1e-5 and
weights max-abs <= 1e-5 (the fast kernels' bar; the generic kernel is tighter).
"""
import numpy as np
import pytest

from oracles import Port, Ref, rel_l2

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
kb = pytest.importorskip("paper_2402_02750_b200")


def draw(rng):
    if rng.random() < 0.5:  # the fast kernels' family
        bits = int(rng.choice([2, 4]))
        G, d = 32, 128
        R = int(rng.choice([32, 64, 128, 256]))
    else:
        bits = int(rng.choice([1, 2, 4, 8]))
        G = int(rng.choice([2, 4, 8, 16, 32]))
        d = G * int(rng.integers(1, max(2, 129 // G)))
        R = G * int(rng.integers(1, 5))
    U = int(rng.integers(1, 6))
    qpk = int(rng.choice([1, 1, 2, 3, 4]))
    l0 = int(rng.integers(1, 3 * R + 300))
    steps = int(rng.integers(1, 5))
    return bits, G, R, d, U, qpk, l0, steps


@pytest.mark.parametrize("case", range(128))
def test_random_shape_vs_reference(cuda, case):
    rng = np.random.default_rng(7000 + case)
    bits, G, R, d, U, qpk, l0, steps = draw(rng)
    ck = Ref() if Ref.available() else Port()
    K = rng.uniform(-1, 1, (U, l0, d)).astype(np.float32)
    V = rng.uniform(-1, 1, (U, l0, d)).astype(np.float32)
    cache = kb.KVCache(kb.CacheConfig(bits, G, R, d), U)
    cache.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
    refs = [[ck.unit(bits, G, R, d) for _ in range(qpk)] for _ in range(U)]
    for u in range(U):
        for r in refs[u]:
            r.prefill(K[u], V[u])
    scale = bool(rng.random() < 0.8)
    where = f"bits={bits} G={G} R={R} d={d} U={U} qpk={qpk} l0={l0}"
    for s in range(steps):
        q = rng.uniform(-1, 1, (U, qpk, d)).astype(np.float32)
        tk = rng.uniform(-1, 1, (U, d)).astype(np.float32)
        tv = rng.uniform(-1, 1, (U, d)).astype(np.float32)
        use_w = s == steps - 1
        res = cache.decode(torch.from_numpy(q).cuda(), torch.from_numpy(tk).cuda(),
                           torch.from_numpy(tv).cuda(), q_per_kv=qpk, weights=use_w,
                           scale_logits=scale)
        out, w = res if use_w else (res, None)
        out = out.cpu().numpy()
        for u in range(U):
            for h in range(qpk):
                ro, rw = refs[u][h].decode(q[u, h], tk[u], tv[u], scale_logits=scale,
                                           weights=True)
                assert rel_l2(out[u, h], ro) <= 1e-5, f"{where} step {s} unit {u} head {h}"
                if use_w:
                    err = float(np.max(np.abs(w[u, h].cpu().numpy() - rw)))
                    assert err <= 1e-5, f"{where} weights {err}"
    torch.cuda.synchronize()
    for u in range(U):
        got, want = cache.export_unit(u), refs[u][0].export()
        for key in want:
            assert got[key].tobytes() == want[key].tobytes(), f"{where} unit {u}: {key}"
    cache.close()
