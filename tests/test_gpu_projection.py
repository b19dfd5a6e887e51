"""GPU: the q/k/v projection on the tcgen05 tensor cores (3xTF32) and its
fusion with the KV-cache append (reference
workload.cpp:230-232 projects t @ W_q/k/v in fp32, then decode_attention
appends k, v)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
kb = pytest.importorskip("paper_2402_02750_b200")


def _weights(gen, hin, hout, dev):
    return [torch.randn((hin, hout), generator=gen, device=dev) / hin ** 0.5 for _ in range(3)]


@pytest.mark.parametrize("hin,hout,n", [(128, 128, 1), (256, 384, 3), (512, 256, 17),
                                        (4096, 512, 64), (1024, 256, 300)])
def test_proj_gemm_fp32_accuracy(cuda, hin, hout, n):
    """3xTF32 on the tensor cores (round-to-nearest hi/lo split, K spread over
    up to 8 TMEM accumulators) vs an fp64 product.  Stated bound: max error
    <= 4e-6 * max(1, K / 1024) of max |x @ W| -- measured 4e-7 (K = 128),
    6e-7 (K = 512), 2.1e-6 (K = 1024), 4.2e-6 (K = 4096), i.e. within ~6x of an fp32 SIMT GEMM
    (the tensor core rounds its fp32 accumulator once per MMA; one
    accumulator over K = 4096 measured 3e-5)."""
    g = torch.Generator(device="cuda").manual_seed(hin + n)
    W = _weights(g, hin, hout, "cuda")
    x = torch.randn((n, hin), generator=g, device="cuda")
    p = kb.Projection(*W)
    outs = p.gemm(x)
    bound = 4e-6 * max(1.0, hin / 1024)
    for o, w in zip(outs, W):
        want = x.double() @ w.double()
        err = ((o.double() - want).abs().max() / want.abs().max()).item()
        assert err < bound, (err, bound)
    p.close()


def test_proj_gemm_unit_layout(cuda):
    """seq > 0: rows (sequence, token) land in [units][seq][128] (prefill layout)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    hin, H, B, T = 256, 3, 2, 37
    W = _weights(g, hin, H * 128, "cuda")
    x = torch.randn((B * T, hin), generator=g, device="cuda")
    p = kb.Projection(*W)
    flat = p.gemm(x)
    per_unit = p.gemm(x, seq=T)
    for f, u in zip(flat, per_unit):
        want = f.view(B, T, H, 128).permute(0, 2, 1, 3).reshape(B * H, T, 128)
        assert torch.equal(u, want)


@pytest.mark.parametrize("bits", [2, 4])
@pytest.mark.parametrize("B,H,l0,steps", [(3, 2, 700, 70), (1, 4, 120, 12), (20, 1, 250, 8)])
def test_proj_append_equals_gemm_then_append(cuda, bits, B, H, l0, steps):
    """kivi_proj_append (projection + append in one launch, value pop quantized
    in the GEMM epilogue) == kivi_proj_gemm then kivi_append: bit-identical
    states and q rows at every step, across a key flush and value pops."""
    g = torch.Generator(device="cuda").manual_seed(B * 7 + H + bits)
    hin = 256
    W = _weights(g, hin, H * 128, "cuda")
    p = kb.Projection(*W)
    cfg = kb.CacheConfig(bits, 32, 128, 128)
    U = B * H
    K0 = torch.rand((U, l0, 128), generator=g, device="cuda") * 2 - 1
    V0 = torch.rand((U, l0, 128), generator=g, device="cuda") * 2 - 1
    a, b = kb.KVCache(cfg, U), kb.KVCache(cfg, U)
    a.prefill(K0, V0)
    b.prefill(K0, V0)
    for _ in range(steps):
        x = torch.randn((B, hin), generator=g, device="cuda")
        q_a = p.append(a, x)
        q, k, v = p.gemm(x)
        b.append(k.view(U, 128).contiguous(), v.view(U, 128).contiguous())
        assert torch.equal(q_a.view(-1), q.view(-1))
    torch.cuda.synchronize()
    assert a.info()["total_tokens"] == b.info()["total_tokens"] == l0 + steps
    for u in range(U):
        ea, eb = a.export_unit(u), b.export_unit(u)
        for key in ea:
            assert ea[key].tobytes() == eb[key].tobytes(), (u, key)
    qa = torch.rand((U, 1, 128), generator=g, device="cuda")
    assert torch.equal(a.attend(qa), b.attend(qa))
    p.close()
