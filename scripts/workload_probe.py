import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2402_02750_b200 as kb
from paper_2402_02750_b200 import workload as wl
from oracles import Ref
sp = wl.WorkloadSpec(batch=3, prompt_len=700, gen_len=5, layers=2, kv_heads=2, head_dim=128)
ref = Ref(); data = ref.workload_data(sp, 3)
want = ref.run_decode_benchmark(sp, 3, 0, 2, 32, 128)
print("reference", want["output_checksum"])
for si in ("0", "1"):
    for vi in ("0", "1"):
        os.environ["KIVI_VIMMA"] = vi; os.environ["KIVI_SMALL_ITEMS"] = si; kb.reload_tuning()
        for fp in (False, True):
            r = wl.run_decode_benchmark(sp, kb.CacheConfig(2, 32, 128, 128), data=data, fused_projection=fp)
            print(f"small_items={si} vimma={vi} fused={fp}: {r.output_checksum:.6f}  rel {(r.output_checksum - want['output_checksum'])/r.output_abs_sum:+.2e}")
