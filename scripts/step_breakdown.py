"""Per-kernel timeline of one C2 layer step in the real pipeline (warm, no
profiler): CUDA events around append, attend and the whole decode."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
dev = torch.device("cuda", 0)
U, D, l0, L = 2048, 128, 4000, 8
cfg = kb.CacheConfig(2, 32, 128, D)
caches = []
kbuf = torch.rand((U, l0, D), device=dev) * 2 - 1
for _ in range(L):
    c = kb.KVCache(cfg, U, capacity_tokens=4300); c.prefill(kbuf, kbuf); caches.append(c)
del kbuf
q = torch.rand((U, 1, D), device=dev); k = torch.rand((U, D), device=dev)
out = torch.empty((U, 1, D), device=dev)
for c in caches: c.decode(q, k, k, out=out)
torch.cuda.synchronize()
def timed(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n): fn(i)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
t_dec = timed(lambda i: caches[i % L].decode(q, k, k, out=out))
t_app = timed(lambda i: caches[i % L].append(k, k))
t_att = timed(lambda i: caches[i % L].attend(q, out=out))
print(f"per layer: decode {t_dec:.1f} us, append {t_app:.1f} us, attend {t_att:.1f} us "
      f"(attend + append = {t_att + t_app:.1f})")
