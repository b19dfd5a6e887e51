"""IMMA value jobs vs CUDA-core value jobs vs the reference, per output."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ["KIVI_SMALL_ITEMS"] = "0"
import paper_2402_02750_b200 as kb
from oracles import Ref, Port
ck = Ref() if Ref.available() else Port()
for U, l0, scale, dist in ((6, 700, 1.0, "normal"), (6, 700, 3.0, "normal"), (16, 1500, 1.0, "uniform")):
    rng = np.random.default_rng(7)
    gen = (lambda *s: rng.standard_normal(s).astype(np.float32) * scale) if dist == "normal" else \
          (lambda *s: rng.uniform(-scale, scale, s).astype(np.float32))
    K, V = gen(U, l0, 128), gen(U, l0, 128)
    q, tk, tv = gen(U, 1, 128), gen(U, 128), gen(U, 128)
    outs = {}
    for vi in ("1", "0"):
        os.environ["KIVI_VIMMA"] = vi
        kb.reload_tuning()
        c = kb.KVCache(kb.CacheConfig(2, 32, 128, 128), U)
        c.prefill(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda())
        outs[vi] = c.decode(torch.from_numpy(q).cuda(), torch.from_numpy(tk).cuda(), torch.from_numpy(tv).cuda()).cpu().numpy()[:, 0]
        c.close()
    want = []
    for u in range(U):
        r = ck.unit(2, 32, 128, 128); r.prefill(K[u], V[u]); want.append(r.decode(q[u, 0], tk[u], tv[u]))
    want = np.array(want)
    for vi, o in outs.items():
        err = o.astype(np.float64) - want
        print(f"U={U} l={l0} {dist}x{scale} VIMMA={vi}: rel-L2 {np.linalg.norm(err)/np.linalg.norm(want):.2e} "
              f"max {np.abs(err).max():.2e} mean signed {err.mean():+.2e} sum diff {err.sum():+.3e} (sum|out| {np.abs(want).sum():.1f})")
