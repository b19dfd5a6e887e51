"""Diagnose the host-buffer (e2e) path: PCIe copy bandwidth, and per-step time
of device-resident decode vs kivi_decode_host, on a reduced C2 (8 layers)."""
import time, torch, numpy as np, sys, os
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
print("is_pinned", h.is_pinned())
L, U, D, ctx = 8, 2048, 128, 4096
cfg = kb.CacheConfig(2, 32, 128, D)
caches = []
kbuf = torch.rand((U, ctx - 300, D), device=dev) * 2 - 1
for _ in range(L):
    c = kb.KVCache(cfg, U, capacity_tokens=ctx + 200); c.prefill(kbuf, kbuf); caches.append(c)
del kbuf
q = torch.rand((L, U, 1, D), device=dev); k = torch.rand((L, U, D), device=dev); v = torch.rand((L, U, D), device=dev)
out = torch.empty((L, U, 1, D), device=dev)
hq, hk, hv = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
ho = torch.empty((L, U, 1, D), pin_memory=True)
def step_dev():
    for ly in range(L): caches[ly].decode(q[ly], k[ly], v[ly], out=out[ly])
def step_host():
    for ly in range(L): caches[ly].decode_host(hq[ly], hk[ly], hv[ly], ho[ly])
for name, fn in (("device", step_dev), ("host", step_host), ("device", step_dev), ("host", step_host)):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); e0.record()
    for _ in range(10): fn()
    t_host = time.perf_counter() - t
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1)/10:.3f} ms/step (GPU events), host enqueue {t_host/10*1e3:.3f} ms/step", flush=True)
