"""Host cost of one decode call (Python wrapper + C-ABI enqueue), C1 shape."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
dev = torch.device("cuda", 0)
U, D, l0 = 32, 128, 4000
c = kb.KVCache(kb.CacheConfig(2, 32, 128, D), U, capacity_tokens=8192)
kbuf = torch.rand((U, l0, D), device=dev)
c.prefill(kbuf, kbuf)
q = torch.rand((U, 1, D), device=dev); k = torch.rand((U, D), device=dev); out = torch.empty((U, 1, D), device=dev)
for _ in range(20): c.decode(q, k, k, out=out)
torch.cuda.synchronize()
n = 200
t = time.perf_counter()
for _ in range(n): c.decode(q, k, k, out=out)
t_enq = (time.perf_counter() - t) / n
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / n
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): c.decode(q, k, k, out=out)
e1.record(); torch.cuda.synchronize()
print(f"decode call: host enqueue {t_enq*1e6:.1f} us, wall per call {t_all*1e6:.1f} us, GPU events per call {e0.elapsed_time(e1)/n*1e3:.1f} us")
# C-ABI only (no Python wrapper): kivi_decode via ctypes directly
f = kb.lib().kivi_decode; s = torch.cuda.current_stream().cuda_stream
args = (c._h, q.data_ptr(), k.data_ptr(), k.data_ptr(), 1, out.data_ptr(), None, 1, s)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(n): f(*args)
print(f"raw ctypes kivi_decode: host enqueue {(time.perf_counter()-t)/n*1e6:.1f} us")
