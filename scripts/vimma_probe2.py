"""IMMA vs CUDA-core value jobs over several decode steps / layers / batches."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KIVI_SMALL_ITEMS"] = "0"
import paper_2402_02750_b200 as kb
for (U, l0, steps, nl) in ((6, 700, 5, 1), (6, 700, 5, 2), (64, 2300, 3, 1)):
    rng = np.random.default_rng(3)
    K = [rng.standard_normal((U, l0, 128)).astype(np.float32) for _ in range(nl)]
    V = [rng.standard_normal((U, l0, 128)).astype(np.float32) for _ in range(nl)]
    qs = [[rng.standard_normal((U, 1, 128)).astype(np.float32) for _ in range(nl)] for _ in range(steps)]
    ks = [[rng.standard_normal((U, 128)).astype(np.float32) for _ in range(nl)] for _ in range(steps)]
    res = {}
    for vi in ("0", "1"):
        os.environ["KIVI_VIMMA"] = vi; kb.reload_tuning()
        cs = []
        for ly in range(nl):
            c = kb.KVCache(kb.CacheConfig(2, 32, 128, 128), U)
            c.prefill(torch.from_numpy(K[ly]).cuda(), torch.from_numpy(V[ly]).cuda()); cs.append(c)
        outs = []
        for s in range(steps):
            for ly in range(nl):
                o = cs[ly].decode(torch.from_numpy(qs[s][ly]).cuda(), torch.from_numpy(ks[s][ly]).cuda(),
                                  torch.from_numpy(ks[s][ly] * 0.7).cuda())
                outs.append(o.cpu().numpy()[:, 0])
        res[vi] = outs
        for c in cs: c.close()
    for i, (a, b) in enumerate(zip(res["0"], res["1"])):
        d = (b.astype(np.float64) - a)
        bad = np.argwhere(np.abs(d) > 1e-4 * np.abs(a).max())
        print(f"U={U} l0={l0} nl={nl} call {i}: rel-L2 {np.linalg.norm(d)/np.linalg.norm(a):.2e} max {np.abs(d).max():.2e} bad {len(bad)} {bad[:6].tolist()}")
