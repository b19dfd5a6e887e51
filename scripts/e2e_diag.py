"""Diagnose the host-buffer (e2e) path: PCIe copy bandwidth, then per-step
GPU-event and wall time of device-resident decode vs kivi_decode_host on a
reduced config (layers x units), stepping l across a 256-token boundary."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
dev = torch.device("cuda", 0)
n = 100 << 20
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty(n // 4, dtype=torch.float32, device=dev)
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize()
    print(f"{name} pinned 100MB: {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s", flush=True)
L = int(os.environ.get("L", 16)); U = int(os.environ.get("U", 1024)); QPK = int(os.environ.get("QPK", 4))
D, ctx = 128, int(os.environ.get("CTX", 8192))
cfg = kb.CacheConfig(2, 32, 128, D)
caches = []
l0 = ctx - 8
kbuf = torch.rand((U, l0, D), device=dev) * 2 - 1
for _ in range(L):
    c = kb.KVCache(cfg, U, capacity_tokens=ctx + 64 + 128); c.prefill(kbuf, kbuf); caches.append(c)
del kbuf
q = torch.rand((L, U, QPK, D), device=dev); k = torch.rand((L, U, D), device=dev); v = torch.rand((L, U, D), device=dev)
out = torch.empty((L, U, QPK, D), device=dev)
hq, hk, hv = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
ho = torch.empty((L, U, QPK, D), pin_memory=True)
def step_dev():
    for ly in range(L): caches[ly].decode(q[ly], k[ly], v[ly], q_per_kv=QPK, out=out[ly])
def step_host():
    for ly in range(L): caches[ly].decode_host(hq[ly], hk[ly], hv[ly], ho[ly], q_per_kv=QPK)
for it in range(12):
    name, fn = ("device", step_dev) if it % 2 == 0 else ("host", step_host)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter(); e0.record()
    fn()
    t_enq = time.perf_counter() - t
    e1.record(); torch.cuda.synchronize()
    print(f"l={caches[0].total_tokens} {name}: {e0.elapsed_time(e1):.3f} ms (GPU events), enqueue {t_enq*1e3:.3f} ms, wall {1e3*(time.perf_counter()-t):.3f} ms", flush=True)
