"""Per-kernel timeline of one layer step in the real pipeline (no profiler):
CUDA events around append, attend (+ combine) and the whole decode.
usage: step_breakdown.py [units=2048] [ctx=4000] [layers=8] [flush=0] [q_per_kv=1]
flush=1 writes 2x L2 between timed calls (each call timed on its own, cold L2),
as bench.py does for states under 4x L2 (C1)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
dev = torch.device("cuda", 0)
U = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
l0 = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
L = int(sys.argv[3]) if len(sys.argv) > 3 else 8
flush = int(sys.argv[4]) if len(sys.argv) > 4 else 0
H = int(sys.argv[5]) if len(sys.argv) > 5 else 1
D = 128
cfg = kb.CacheConfig(2, 32, 128, D)
caches = []
kbuf = torch.rand((U, l0, D), device=dev) * 2 - 1
for _ in range(L):
    c = kb.KVCache(cfg, U, capacity_tokens=l0 + 300); c.prefill(kbuf, kbuf); caches.append(c)
del kbuf
q = torch.rand((U, H, D), device=dev); k = torch.rand((U, D), device=dev)
out = torch.empty((U, H, D), device=dev)
for c in caches: c.decode(q, k, k, q_per_kv=H, out=out)
torch.cuda.synchronize()
scratch = torch.empty(2 * (126 << 20) // 4, device=dev) if flush else None
def timed(fn, n=20):
    if not flush:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n): fn(i)
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3
    tot = 0.0
    for i in range(n):
        scratch.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(i); e1.record(); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3
t_dec = timed(lambda i: caches[i % L].decode(q, k, k, q_per_kv=H, out=out))
t_app = timed(lambda i: caches[i % L].append(k, k))
t_att = timed(lambda i: caches[i % L].attend(q, q_per_kv=H, out=out))
print(f"U={U} H={H} l={l0} flush={flush}: decode {t_dec:.1f} us, append {t_app:.1f} us, attend {t_att:.1f} us "
      f"(attend + append = {t_att + t_app:.1f})")
# attend kernels alone (library events around the attend launches, no combine)
for c in caches:
    c.profile_read(); c.profile_enable(True)
t_att2 = timed(lambda i: caches[i % L].attend(q, q_per_kv=H, out=out))
ms, n = 0.0, 0
for c in caches:
    m_, n_, _ = c.profile_read(); ms += m_; n += n_
    c.profile_enable(False)
print(f"  attend kernels {ms / max(n, 1) * 1e3:.1f} us of attend() {t_att2:.1f} us "
      f"(combine + gaps {t_att2 - ms / max(n, 1) * 1e3:.1f} us)")
