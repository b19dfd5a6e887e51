"""Small decodes through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on the GPU box:
    compute-sanitizer --tool racecheck python scripts/sanitize_decode.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(5)


def run(bits, U, l0, qpk, path, steps=3, small="0"):
    os.environ["KIVI_SMALL_ITEMS"] = small
    d = 128
    c = kb.KVCache(kb.CacheConfig(bits, 32, 128, d), U)
    c.set_attend_path(path)
    K = torch.rand((U, l0, d), device=dev, generator=g) * 2 - 1
    c.prefill(K, K.flip(1).contiguous())
    for _ in range(steps):
        q = torch.rand((U, qpk, d), device=dev, generator=g)
        k = torch.rand((U, d), device=dev, generator=g)
        out = c.decode(q, k, k, q_per_kv=qpk)
    torch.cuda.synchronize()
    c.close()
    return float(out.abs().sum())


for args in [(2, 16, 700, 1, "fast"), (4, 8, 700, 1, "fast"), (2, 8, 1100, 4, "fast"),
             (2, 8, 1100, 2, "fast"), (2, 4, 300, 1, "generic"), (2, 4, 383, 1, "fast", 3, "1"),
             (2, 4, 127, 4, "fast")]:
    print(args, run(*args), flush=True)
# projection on tcgen05 fused with the append (K8), across a key-tile boundary
hin, H, B = 256, 2, 3
c = kb.KVCache(kb.CacheConfig(2, 32, 128, 128), B * H)
Kp = torch.rand((B * H, 95, 128), device=dev, generator=g) * 2 - 1
c.prefill(Kp, Kp)
W = [torch.randn((hin, H * 128), device=dev, generator=g) / hin ** 0.5 for _ in range(3)]
p = kb.Projection(*W)
for _ in range(3):
    x = torch.randn((B, hin), device=dev, generator=g)
    q = p.append(c, x)
    out = c.attend(q)
p.gemm(torch.randn((5, hin), device=dev, generator=g))
torch.cuda.synchronize()
print("projection", float(out.abs().sum()), flush=True)
p.close()
c.close()

# single-layer host step: k / v read from mapped pinned memory, q staged by the
# append warps (QStage), outputs written back across PCIe
U = 8
c = kb.KVCache(kb.CacheConfig(2, 32, 128, 128), U)
Kh = torch.rand((U, 300, 128), device=dev, generator=g)
c.prefill(Kh, Kh)
st = kb.LayerStack([c])
hq, hk, hv, ho = (torch.rand(sh).pin_memory() for sh in ((1, U, 1, 128), (1, U, 128), (1, U, 128),
                                                         (1, U, 1, 128)))
for _ in range(3):
    st.decode_host(hq, hk, hv, ho)
print("host step", float(ho.abs().sum()), flush=True)
c.close()
print("sanitize run done")
