"""Generates tests/golden/workload_golden.json (+ workload_tiny.npz) from the
REFERENCE itself (oracle/_ref/ref_cbridge.so: reference workload.cpp compiled by
oracle/Makefile).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_workload_golden.py

Pins the workload layer: estimate_memory / max_batch_at_budget on the presets and
a grid of specs, and one tiny run_decode_benchmark (its exact synthetic data and
the reference's checksum and peak bytes) for the GPU driver's parity test.
"""
import json
import os
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import Ref  # noqa: E402


@dataclass
class S:
    batch: int = 1
    prompt_len: int = 161
    gen_len: int = 338
    layers: int = 2
    kv_heads: int = 2
    head_dim: int = 64


SPECS = [S(512, 512, 32, 96, 96, 128), S(16, 3968, 128, 32, 32, 128), S(),
         S(3, 100, 29, 2, 4, 64), S(1, 127, 1, 1, 1, 32), S(7, 128, 0, 3, 2, 32),
         S(2, 4000, 96, 32, 32, 128), S(1, 1, 1, 1, 1, 8)]
CFGS = [(2, 32, 128), (4, 32, 128), (2, 8, 32), (8, 4, 8), (1, 8, 16)]
TINY = (S(2, 40, 6, 2, 2, 32), 2, 32, 32, 11)   # spec, bits, G, R, seed


def main():
    ref = Ref()
    est = []
    for sp in SPECS:
        for bits, G, R in CFGS:
            if sp.head_dim % G or R % G:
                continue
            est.append({"spec": list(vars(sp).values()), "cfg": [bits, G, R],
                        **ref.estimate_memory(sp, bits, G, R)})
    mb = []
    for sp in (S(1, 2048, 0, 32, 32, 128), S(1, 512, 32, 96, 96, 128), S(1, 161, 338, 2, 2, 64)):
        for budget in (80 << 30, 24 << 30, 1 << 30, 123456789):
            for fp_mode in (0, 1):
                try:
                    b = ref.max_batch_at_budget(sp, budget, fp_mode, 2, 32, 128)
                except Exception as e:  # BudgetError
                    b = -1
                mb.append({"spec": list(vars(sp).values()), "budget": budget,
                           "mode": "fp" if fp_mode else "kivi", "batch": b})
    sp, bits, G, R, seed = TINY
    w, pr, tk = ref.workload_data(sp, seed)
    runs = {}
    for fp_mode in (0, 1):
        runs["fp" if fp_mode else "kivi"] = ref.run_decode_benchmark(sp, seed, fp_mode, bits, G, R)
    np.savez_compressed(os.path.join(HERE, "workload_tiny.npz"), weights=w, prompts=pr, tokens=tk)
    with open(os.path.join(HERE, "workload_golden.json"), "w") as f:
        json.dump({"generator": "oracle/_ref (reference workload.cpp)", "estimate_memory": est,
                   "max_batch_at_budget": mb,
                   "tiny_run": {"spec": list(vars(sp).values()), "cfg": [bits, G, R],
                                "seed": seed, "reference": runs}}, f, indent=1)
    print(len(est), "estimates,", len(mb), "budgets, tiny run", runs)


if __name__ == "__main__":
    main()
