"""Native driver failure isolation."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_02750_b200 as kb
from paper_2402_02750_b200 import workload as wl
cfg = kb.CacheConfig(2, 32, 128, 128)
for (b, P, g, L, H, devs) in ((5, 260, 9, 2, 2, (0,)), (5, 260, 9, 2, 2, (0, 0)), (3, 700, 5, 2, 2, (0,)),
                              (4, 256, 4, 1, 2, (0,)), (5, 256, 4, 1, 2, (0,)), (5, 260, 4, 1, 1, (0,))):
    sp = wl.WorkloadSpec(batch=b, prompt_len=P, gen_len=g, layers=L, kv_heads=H, head_dim=128)
    try:
        r = wl.run_decode_benchmark_native(sp, cfg, seed=11, devices=devs)
        print("OK ", (b, P, g, L, H, devs), r.output_checksum, r.peak_cache_bytes)
    except Exception as e:
        print("ERR", (b, P, g, L, H, devs), type(e).__name__, e)
