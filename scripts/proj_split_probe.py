"""Accuracy of the tcgen05 3xTF32 projection per split mode (KIVI_PROJ_SPLIT)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
for mode in ("0", "1", "2"):
    os.environ["KIVI_PROJ_SPLIT"] = mode
    kb.reload_tuning()
    for hin, hout, n in ((128, 128, 1), (512, 256, 17), (4096, 512, 64)):
        g = torch.Generator(device="cuda").manual_seed(hin + n)
        W = [torch.randn((hin, hout), generator=g, device="cuda") / hin ** 0.5 for _ in range(3)]
        x = torch.randn((n, hin), generator=g, device="cuda")
        p = kb.Projection(*W)
        outs = p.gemm(x)
        errs = []
        for o, w in zip(outs, W):
            want = x.double() @ w.double()
            errs.append(((o.double() - want).abs().max() / want.abs().max()).item())
        f32 = ((x @ W[0]).double() - x.double() @ W[0].double()).abs().max().item() / (x.double() @ W[0].double()).abs().max().item()
        print(f"split={mode} K={hin:5d} N={n:3d}: rel err q/k/v {errs[0]:.2e} {errs[1]:.2e} {errs[2]:.2e}  (fp32 SIMT {f32:.2e})")
        p.close()
