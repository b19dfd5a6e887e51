import os, sys
sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo")
import test_gpu_parity as t
import paper_2402_02750_b200 as kb
for item in os.environ.get("ITEMS", "256 384").split():
    os.environ["KIVI_GQA_ITEM"] = item
    kb.reload_tuning()
    for qpk in (2, 4):
        for seedcase in [(1.0, 1.0, 1.0, (1, 17, 40)), (1.0, 1.0, 1.0, ())]:
            ks, vs, qs, outl = seedcase
            for seed in (0, 1, 2):
                e, ew = t.run_gqa((2, 32, 128, 128), U=3, qpk=qpk, l0=1100, steps=2, path="fast",
                                  seed=int(ks * 10 + vs) + qpk + 100 * seed, weights=True, kscale=ks,
                                  vscale=vs, qscale=qs, outliers=outl)
                print(item, qpk, outl, seed, f"{e:.3g} {ew:.3g}", flush=True)
