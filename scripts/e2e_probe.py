"""Where the C1 end-to-end step goes (host buffers, one layer, 32 units)."""
import ctypes, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
dev = torch.device("cuda", 0)
U, D, l0, n = 32, 128, 3900, 100
c = kb.KVCache(kb.CacheConfig(2, 32, 128, D), U, capacity_tokens=8192)
kbuf = torch.rand((U, l0, D), device=dev)
c.prefill(kbuf, kbuf)
st = kb.LayerStack([c])
s = torch.cuda.Stream()
hq, hk, hv, ho = (torch.rand(sh).pin_memory() for sh in ((1, U, 1, D), (1, U, D), (1, U, D), (1, U, 1, D)))
def timeit(f, label):
    for _ in range(10): f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    print(f"{label:50s} {(time.perf_counter() - t) / n * 1e6:7.1f} us/step")
for zc in ("65536", "0"):
    os.environ["KIVI_ZERO_COPY_BYTES"] = zc
    kb.lib().kivi_reload_tuning()
    timeit(lambda: st.decode_host(hq, hk, hv, ho, stream=s), f"LayerStack.decode_host zero_copy={zc}")
    f = kb.lib().kivi_decode_layers_host
    args = (st._arr, 1, hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), 1, ho.data_ptr(), 1, s.cuda_stream)
    timeit(lambda: f(*args), f"raw ctypes kivi_decode_layers_host zero_copy={zc}")
dq, dk, dv, do = (x.cuda() for x in (hq, hk, hv, ho))
def devstep():
    st.decode(dq, dk, dv, do)
    torch.cuda.current_stream().synchronize()
timeit(devstep, "device rows decode + stream sync")
def devnosync():
    st.decode(dq, dk, dv, do)
timeit(devnosync, "device rows decode, no sync (pipelined)")
def cp():
    dq.copy_(hq, non_blocking=True); torch.cuda.current_stream().synchronize()
timeit(cp, "16 KB H2D copy + sync")
def sync_only():
    torch.cuda.current_stream().synchronize()
timeit(sync_only, "empty stream sync")
