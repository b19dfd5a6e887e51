import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_parity as t
import paper_2402_02750_b200 as kb
def probe(qpk, ks, vs, qs, outl, voutl=(), l0=1100, seed=5):
    ck = t.checker(); rng = np.random.default_rng(seed); cfg = (2, 32, 128, 128); U = 2; d = 128
    K, V = t.rnd(rng, U, l0, d, scale=ks), t.rnd(rng, U, l0, d, scale=vs)
    for c in outl: K[:, :, c] *= 50
    for c in voutl: V[:, :, c] *= 50
    cache = kb.KVCache(kb.CacheConfig(*cfg), U); cache.set_attend_path("fast"); cache.prefill(t.dev(K), t.dev(V))
    refs = [[ck.unit(*cfg) for _ in range(qpk)] for _ in range(U)]
    for u in range(U):
        for h in range(qpk): refs[u][h].prefill(K[u], V[u])
    q = t.rnd(rng, U, qpk, d, scale=qs); tk, tv = t.rnd(rng, U, d, scale=ks), t.rnd(rng, U, d, scale=vs)
    for c in outl: tk[:, c] *= 50
    for c in voutl: tv[:, c] *= 50
    out, w = cache.decode(t.dev(q), t.dev(tk), t.dev(tv), q_per_kv=qpk, weights=True)
    out = out.cpu().numpy(); w = w.cpu().numpy()
    eo, ew, el = 0, 0, 0
    for u in range(U):
        for h in range(qpk):
            ro, rw = refs[u][h].decode(q[u, h], tk[u], tv[u], weights=True)
            eo = max(eo, t.rel_l2(out[u, h], ro)); ew = max(ew, np.max(np.abs(w[u, h] - rw)))
            m = rw > 1e-6
            dl = np.log2(w[u, h][m]) - np.log2(rw[m]); el = max(el, np.std(dl) if m.sum() > 1 else 0)
            rng_l = np.log2(rw[m].max() / rw[m].min()) if m.sum() > 1 else 0
    print(f"qpk={qpk} ks={ks} vs={vs} qs={qs} ko={outl} vo={voutl}: out {eo:.3g} w {ew:.3g} dlogit_std {el:.3g} (log2 range {rng_l:.1f})", flush=True)
for qpk in (2, 4):
    probe(qpk, 1, 1, 1, ())
    probe(qpk, 1, 1, 1, (1, 17, 40))
    probe(qpk, 1, 1, 20, ())
    probe(qpk, 1, 1, 1, (), (1, 17, 40))
    probe(qpk, 4, 0.01, 20, (5,))
