#!/usr/bin/env python3
"""bench.py — KIVI 2-bit fused dequant-attention decode on B200.

One "step" = one decode step of the whole model over one batch: for every
layer, append the new token's K/V to every (batch, kv-head) unit and attend
with the new query (reference decode_attention, attention.cpp:26-100, driven
the way run_decode_benchmark drives it, workload.cpp:224-242).

Default workload = BASELINE.json configs[1] (C2): Llama-2-7B, 32 layers x 32
kv-heads, head_dim 128, batch 64 per GPU, ctx 4096, 2-bit, G=32, R=128.  The
state is prefilled on the device to ctx - warmup - steps tokens so the last
timed step ends at l = ctx.  The 38 GB state is far larger than the 126 MB L2,
so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference]

Under torchrun (N > 1) every rank runs the same per-GPU workload on its own
device (weak scaling over batch: the units shard with no collective); times
are max-reduced over ranks with NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn tokens/s and achieved HBM GB/s vs roofline, 1/2/4/8 B200"
OUTLIER_CHANNELS = [1, 17, 40]  # analysis.hpp:59-61


def data_note(args):
    dist = "N(0,1)" if args.data == "normal" else "uniform(-1,1)"
    out = ", key channels {1,17,40} x50" if args.outliers else ""
    return f"synthetic ({dist} K/V/q{out}, generated on device; random-init, no checkpoint)"

# name -> (layers, kv_heads, batch, ctx, bits, q_per_kv, description)
CONFIGS = {
    "c1": (1, 32, 1, 4096, 2, 1, "single layer, 32 heads, head_dim=128, batch 1, ctx 4096, 2-bit"),
    "c2": (32, 32, 64, 4096, 2, 1, "Llama-2-7B all 32 layers decode, batch 64, ctx 4096, 2-bit"),
    "c3": (32, 8, 128, 8192, 2, 4, "Mistral-7B GQA (8 kv-heads, 4 q/kv), batch 128, ctx 8192, 2-bit"),
    "c4": (40, 40, 256, 4096, 2, 1, "Llama-2-13B decode, batch 256, ctx 4096, 2-bit"),
    "c5": (32, 32, 16, 32768, 2, 1, "Llama-2-7B shape, batch 16, ctx 32768, 2-bit"),
}
G, R, D = 32, 128, 128


def attend_bytes_per_unit(l, bits, qpk=1, d=D, g=G, r=R):
    """SURVEY §8d algorithmic bytes of one unit's attend (reads + q/out)."""
    kr = l % r
    kg = l - kr
    vr = min(l, r)
    vg = l - vr
    return ((kg * d * bits + 7) // 8 + (vg * d * bits + 7) // 8 + (kg * d // g + vg * d // g) * 8
            + (kr + vr) * d * 4 + qpk * d * 8)


def state_bytes_per_unit(capacity, bits, layers, d=D, g=G, r=R):
    """Device bytes of one (batch, kv-head) unit over all layers: code streams,
    (lo, hi) pairs and the two fp32 residual rings."""
    cap = -(-capacity // r) * r
    codes = 2 * cap * d * bits // 8
    pairs = 2 * (cap // g) * d * 8
    rings = 2 * r * d * 4
    return layers * (codes + pairs + rings + 4 * 256)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.idx, self.period = device_index, period_s
        self.pci = None
        try:
            import torch
            p = torch.cuda.get_device_properties(device_index)
            self.pci = "%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        except Exception:
            pass
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            try:
                self.h = nv.nvmlDeviceGetHandleByPciBusId(self.pci)
            except Exception:
                self.h = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover - NVML absent
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown",
                                               0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for n, bit in names.items():
                    if mask & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def clocks_bad(cs):
    """A timed region's clock summary that rejects the measurement: a hardware
    or thermal slowdown, or SM clocks stuck well below max with no reason (a
    leftover clock lock).  sw_power_cap is kept (noted in the line)."""
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if set(cs.get("reasons") or []) & bad:
        return True
    mhz, mx = cs.get("sm_mhz"), cs.get("sm_max_mhz")
    return bool(mhz and mx and mhz < 0.75 * mx and not cs.get("reasons"))


def attend_kernel_name(qpk, units, ctx, sms=148):
    """The attend launch the roofline times (library routing, kivi_b200.cu)."""
    if qpk > 1:
        return ("kivi_b200::gqa_tc::attend_gqa_tc_kernel (tensor cores) + "
                "gqa::attend_gqa_kernel (residual items, side stream)")
    if units * -(-ctx // 256) < 4 * sms:
        return "kivi_b200::fast::attend_tail_kernel (few-unit route, short items)"
    return ("kivi_b200::fast::attend_body_kernel + attend_tail_kernel (concurrent, one stream, "
            "programmatic launch)")


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def self_launch(n):
    """`bench.py --gpus N` outside torchrun: re-runs this command as N ranks
    (one process per GPU) through torch.distributed.run on 127.0.0.1 and
    returns its exit code.  NCCL logs (NCCL_DEBUG=INFO unless set) go to
    gpurun_out/nccl.<host>.<pid>.log so stdout keeps rank 0's one JSON line."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    if "NCCL_DEBUG_FILE" not in env:
        logdir = os.path.join(ROOT, "gpurun_out")
        os.makedirs(logdir, exist_ok=True)
        env["NCCL_DEBUG_FILE"] = os.path.join(logdir, "nccl.%h.%p.log")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def workload_config(args, world, rank=0, free_bytes=None):
    """The workload both arms report (same keys, same values): BASELINE config,
    per-GPU units, scaling mode and, when a rank's share does not fit its HBM,
    the largest power-of-two batch that does (C4 on one GPU)."""
    from paper_2402_02750_b200.sharding import partition_units
    layers, heads, batch, ctx, bits, qpk, desc = CONFIGS[args.config]
    if args.layers:
        layers = args.layers
    if args.bits:
        bits = args.bits
        desc = desc.replace("2-bit", f"{bits}-bit")
    scaling = args.scaling or ("strong" if args.config in ("c4", "c5") else "weak")
    if scaling == "strong":
        U = len(partition_units(batch, heads, world, rank))  # fixed global batch
        global_batch = batch
    else:
        U = batch * heads  # every rank serves its own batch
        global_batch = batch * world
    steps, warmup = args.steps, args.warmup
    capacity_note = None
    per_unit = state_bytes_per_unit(ctx + steps + warmup + R, bits, layers) + 2 * 4 * D * ctx
    if free_bytes is not None and U * per_unit > 0.85 * free_bytes:
        b_rank = max(1, U // heads)
        while b_rank > 1 and b_rank * heads * per_unit > 0.85 * free_bytes:
            b_rank //= 2
        capacity_note = (f"{U // heads} sequences/GPU need {U * per_unit / 1e9:.0f} GB of "
                         f"state > {free_bytes / 1e9:.0f} GB free: timed {b_rank} sequences/GPU")
        U = b_rank * heads
        global_batch = b_rank * world
        scaling = "weak"
    cfg = {"workload": desc, "name": args.config, "layers": layers, "kv_heads": heads,
           "batch_per_gpu": global_batch / world, "global_batch": global_batch, "ctx": ctx,
           "bits": bits, "group_size": G, "residual": R, "head_dim": D, "q_per_kv": qpk,
           "units_per_layer_per_gpu": U, "capacity_limited": capacity_note,
           "l_timed": [ctx - steps + 1, ctx],
           "parallelism": f"dp{world} ({scaling}; units sharded by (batch, kv-head), "
                          "no collective)"}
    return cfg, U, scaling


# ---- the reference / oracle legs (the only code here that executes oracle/) --

def cpu_reference_sample(cfg_name, steps, warmup, threads, units=None, bits=0):
    """Times the REFERENCE decode_attention (oracle/_ref, compiled from the
    reference sources) on a bounded sample of the workload's units; returns
    (unit-steps per second, description, kind, measured seconds, units)."""
    layers, heads, batch, ctx, cbits, qpk, _ = CONFIGS[cfg_name]
    bits = bits or cbits
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref
    if not Ref.available():
        raise RuntimeError("oracle/_ref/ref_cbridge.so missing (build with make -C oracle)")
    units = units or max(threads * 2, 16)
    l0 = max(1, ctx - warmup - steps)
    secs, _ = Ref().bench_decode(bits, G, R, D, units, l0, warmup, steps, threads, seed=11)
    rate = units * steps / secs  # unit-steps / s (each = one reference decode_attention call)
    desc = (f"{units} units x {steps} timed decode steps (after {warmup} warm-up) at l={l0}.."
            f"{l0 + warmup + steps}, reference decode_attention per unit (append+attend), "
            f"{threads} threads, {secs:.2f} s measured; extrapolated linearly to "
            f"{layers * heads * batch * qpk} unit-steps/step")
    return rate, desc, "reference", secs, units


def reference_parity_sample(bits, qpk, prompts, seq, outs, states):
    """Replays the sampled units of layer 0 through the reference itself
    (oracle/_ref: prefill, append_token per step, decode_attention on the last
    one, per query head on a state copy) and compares with what the timed GPU
    path produced: the exported state bit-exactly, the last output by rel-L2.
    prompts: {unit: (K, V)}; seq: [(k[U,d], v[U,d], q[U,qpk,d])] per step;
    outs: {unit: [qpk, d]} last-step outputs; states: {unit: exported state}."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref, rel_l2
    if not Ref.available():
        return None
    ref = Ref()

    def one(u):
        K, V = prompts[u]
        r = ref.unit(bits, G, R, D)
        r.prefill(K, V)
        for tk, tv, _ in seq[:-1]:
            r.append(tk[u], tv[u])
        tk, tv, q = seq[-1]
        heads = [r] + [r.clone() for _ in range(qpk - 1)]
        err = 0.0
        for h in range(qpk):
            err = max(err, rel_l2(outs[u][h], heads[h].decode(q[u, h], tk[u], tv[u])))
        want = r.export()
        exact = all(np.asarray(states[u][k]).tobytes() == want[k].tobytes() for k in want)
        return err, exact

    with ThreadPoolExecutor(max_workers=len(prompts)) as ex:
        res = list(ex.map(one, sorted(prompts)))
    return {"units": sorted(int(u) for u in prompts), "layer": 0,
            "checker": "reference (oracle/_ref)",
            "steps_replayed": len(seq), "state_bit_exact": all(e for _, e in res),
            "max_rel_l2": max(e for e, _ in res), "bar_rel_l2": 1e-5}


def run_reference_arm(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    world = max(world, args.gpus)
    cfg, _, scaling = workload_config(args, world, 0, None)
    layers, heads, qpk, bits = cfg["layers"], cfg["kv_heads"], cfg["q_per_kv"], cfg["bits"]
    batch = cfg["global_batch"]
    threads = os.cpu_count() or 1
    # each "step" is a bounded sample: ~16 units per thread, one decode each
    rate, sample, kind, secs, units = cpu_reference_sample(args.config, args.steps, args.warmup,
                                                           threads, units=16 * threads, bits=bits)
    unit_steps_per_step = layers * heads * batch * qpk
    step_s = unit_steps_per_step / rate  # a full step of the workload, extrapolated
    tok_s = batch / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        # the timed step IS the bounded sample: its measured duration
        "ms_per_step": secs / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None, "dtype": "f32/f64 (reference CPU)",
        "data": "synthetic (uniform(-1,1) from the oracle's counter RNG; CPU time is data-independent)",
        "config": cfg,
        "sampled_units": units, "sample_seconds": secs,
        "ms_per_full_step_extrapolated": step_s * 1e3,
        "ms_per_step_note": (f"each timed step is a bounded sample: {units} of the "
                             f"{unit_steps_per_step} reference decode_attention calls of a "
                             f"full step ({args.steps} steps measured in {secs:.2f} s); value "
                             "= the sample's tokens-equivalent rate"),
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_dry(args):
    """CPU rehearsal of the multi-rank path (gloo, no GPU): every rank takes its
    unit shard, 'times' it, and the max over ranks is reduced; rank 0 prints the
    JSON line.  Covered by tests/test_bench_launch.py through self_launch."""
    import torch.distributed as dist
    world, rank, _ = dist_setup()
    if world > 1:
        dist.init_process_group("gloo")
    cfg, U, scaling = workload_config(args, world, rank, None)
    t = 1e-3 * (1 + rank)
    from paper_2402_02750_b200.sharding import max_over_ranks
    t = max_over_ranks(t)
    units = [U]
    if world > 1:
        units = [None] * world
        dist.all_gather_object(units, U)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "value": None,
                          "unit": "tokens/s", "steps": args.steps, "warmup": args.warmup,
                          "scaling": scaling, "config": cfg, "units_per_rank": units,
                          "max_rank_time_s": t}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def percentiles(xs):
    ys = sorted(xs)
    if not ys:
        return None

    def p(f):
        return ys[min(len(ys) - 1, max(0, int(math.ceil(f * len(ys))) - 1))]

    # at_ctx: the last timed step, the one at l = ctx
    return {"p50": p(0.5), "p90": p(0.9), "p99": p(0.99), "max": ys[-1],
            "mean": sum(ys) / len(ys), "n": len(ys), "at_ctx": xs[-1]}


def run_ours(args):
    import numpy as np
    import torch
    import paper_2402_02750_b200 as kb

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    free, _ = torch.cuda.mem_get_info(dev)
    config, U, scaling = workload_config(args, world, rank, free)
    layers, heads, ctx, bits, qpk = (config["layers"], config["kv_heads"], config["ctx"],
                                     config["bits"], config["q_per_kv"])
    global_batch = int(config["global_batch"])
    steps, warmup = args.steps, args.warmup
    l0 = ctx - warmup - steps
    if l0 < 1:
        raise SystemExit("--steps + --warmup must be < ctx")
    cfg = kb.CacheConfig(bits, G, R, D)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- state: prefilled on the device; rebuilt identically before each pass
    caches = [kb.KVCache(cfg, U, capacity_tokens=ctx + steps + warmup + R, device=local)
              for _ in range(layers)]
    for c in caches:
        c.set_attend_path("auto")
    kbuf = torch.empty((U, l0, D), device=dev, dtype=torch.float32)
    vbuf = torch.empty_like(kbuf)
    gen = torch.Generator(device=dev)
    do_parity = rank == 0 and world == 1 and not args.no_cpu_baseline and not args.no_parity
    sample_units = sorted({(i * U) // 8 + (i % 3) for i in range(8)} & set(range(U)))
    prompts = {}

    def fill(t, keys=False):
        """SURVEY §8d inputs: N(0, 1) (or uniform(-1, 1)); --outliers scales key
        channels {1, 17, 40} by 50 (analysis.hpp:59-61): scales change, bytes do not."""
        if args.data == "normal":
            t.normal_(0.0, 1.0, generator=gen)
        else:
            t.uniform_(-1.0, 1.0, generator=gen)
        if keys and args.outliers:
            t[..., OUTLIER_CHANNELS] *= 50.0
        return t

    def rebuild():
        """Every layer back to l0 tokens, from the same seeded draws."""
        for ly in range(layers):
            gen.manual_seed(1234 + 1000 * rank + ly)
            fill(kbuf, keys=True)
            fill(vbuf)
            caches[ly].prefill(kbuf, vbuf)
            if ly == 0 and do_parity and not prompts:
                for u in sample_units:
                    prompts[u] = (kbuf[u].cpu().numpy(), vbuf[u].cpu().numpy())
        torch.cuda.synchronize()

    # per-step inputs resident in HBM (a pool of 2 sets per layer, cycled)
    pool = 2
    gen.manual_seed(99 + rank)
    qs = fill(torch.empty((pool, layers, U, qpk, D), device=dev))
    ks = fill(torch.empty((pool, layers, U, D), device=dev), keys=True)
    vs = fill(torch.empty((pool, layers, U, D), device=dev))
    outs = torch.empty((layers, U, qpk, D), device=dev)

    stack = kb.LayerStack(caches)  # one C-ABI call per step: the layer loop is native

    def step(j):
        p = j % pool
        stack.decode(qs[p], ks[p], vs[p], outs, q_per_kv=qpk)

    # A state smaller than 4x L2 (C1: 18.6 MB vs 126 MB) would be served from
    # L2: then every timed step is bracketed by its own events and L2 is
    # flushed (a 2x-L2 write) between steps, outside the events.
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    state_total = U * state_bytes_per_unit(ctx + steps + warmup + R, bits, layers)
    flush = state_total < 4 * l2
    scratch = torch.empty((2 * l2) // 4, dtype=torch.float32, device=dev) if flush else None
    l2_note = (f"state {state_total / 1e6:.1f} MB < 4x L2 ({l2 >> 20} MB): L2 flushed by a "
               f"{2 * l2 >> 20} MB write between timed steps (per-step events)" if flush else
               f"state {state_total / 1e9:.1f} GB >> {l2 >> 20} MB L2 (inputs larger than L2, "
               "no flush)")

    def timed_steps(per_step_events):
        """K timed steps after W warm-up ones; returns (total s, per-step ms)."""
        for j in range(warmup):
            step(j)
        barrier()
        if per_step_events or flush:
            evs = []
            for i in range(steps):
                if flush:
                    scratch.fill_(float(i))
                a_ = torch.cuda.Event(enable_timing=True)
                b_ = torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                step(warmup + i)
                b_.record(stream)
                evs.append((a_, b_))
            barrier()
            per = [a_.elapsed_time(b_) for a_, b_ in evs]
            return sum(per) / 1e3, per
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            step(warmup + i)
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1) / 1e3, None

    # ---- pass A: `value` (nothing recorded inside the timed region but the two
    # events bracketing it; launches counted by the library on the host)
    rebuild()
    for c in caches:
        c.profile_read()
    with ClockSampler(local) as clocks:
        elapsed_local, per_a = timed_steps(False)
    elapsed = max_over_ranks(elapsed_local)
    # A timed region that saw a hardware / thermal slowdown, or SM clocks stuck
    # well below max with no reason (a leftover clock lock), is re-measured
    # once (any rank's verdict applies to all); the first attempt is reported.
    remeasured = None
    if max_over_ranks(float(clocks_bad(clocks.summary()))) > 0:
        remeasured = {"first_value": global_batch * steps / elapsed,
                      "first_clocks": clocks.summary()}
        rebuild()
        for c in caches:
            c.profile_read()  # launches are counted over the re-measured pass only
        with ClockSampler(local) as clocks:
            elapsed_local, per_a = timed_steps(False)
        elapsed = max_over_ranks(elapsed_local)
    launches = 0
    for c in caches:
        launches += c.profile_read()[2]
    launches = launches * steps // (steps + warmup)  # the timed steps' share (same per step)
    tok_s = global_batch * steps / elapsed
    ms_per_step = elapsed / steps * 1e3

    # ---- pass B: step-latency distribution (an event pair per step)
    if per_a is None:
        rebuild()
        _, per_b = timed_steps(True)
    else:
        per_b = per_a
    latency = percentiles(per_b)

    # ---- pass C: the attend launch alone (events around every attend launch),
    # for the roofline; not part of `value`
    rebuild()
    for j in range(warmup):
        step(j)
    barrier()
    for c in caches:
        c.profile_read()
        c.profile_enable(1)
    for i in range(steps):
        if flush:
            scratch.fill_(float(i))
        step(warmup + i)
    barrier()
    kern_ms, kern_n = 0.0, 0
    for c in caches:
        ms, n, _ = c.profile_read()
        kern_ms += ms
        kern_n += n
        c.profile_enable(False)
    alg_bytes = sum(attend_bytes_per_unit(l0 + warmup + i + 1, bits, qpk) for i in range(steps))
    alg_bytes *= U * layers
    per_launch_bytes = alg_bytes / (steps * layers)
    avg_launch_s = max_over_ranks((kern_ms / 1e3) / max(kern_n, 1))
    achieved = per_launch_bytes / avg_launch_s / 1e9 if avg_launch_s > 0 else float("nan")
    peak, peak_src = load_peaks()

    # ---- pass D: e2e through the C-ABI host-buffer entry point, same window ---
    e2e = None
    seq_used = None
    last_out = None
    if not args.no_e2e:
        hq = torch.empty((pool, layers, U, qpk, D), dtype=torch.float32, pin_memory=True)
        hk = torch.empty((pool, layers, U, D), dtype=torch.float32, pin_memory=True)
        hv = torch.empty((pool, layers, U, D), dtype=torch.float32, pin_memory=True)
        ho = torch.empty((layers, U, qpk, D), dtype=torch.float32, pin_memory=True)
        hq.copy_(qs.cpu())
        hk.copy_(ks.cpu())
        hv.copy_(vs.cpu())

        # a stream of its own (a CUDA graph cannot capture the legacy default stream)
        e2e_stream = torch.cuda.Stream(device=dev)

        # uploads, every layer, the result copy; each call returns with the
        # outputs on the host (the next step's inputs would depend on them).
        # One bound call per pool slot: the pinned buffers are fixed, as in a
        # serving loop that refills them every step.
        bound = [stack.bind_host_step(hq[p], hk[p], hv[p], ho, q_per_kv=qpk, stream=e2e_stream)
                 for p in range(pool)]

        def host_step(j):
            bound[j % pool]()

        rebuild()
        for j in range(warmup):
            host_step(j)
        barrier()
        t0 = time.perf_counter()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(e2e_stream)
        for i in range(steps):
            host_step(warmup + i)
        f1.record(e2e_stream)
        barrier()
        wall = time.perf_counter() - t0
        e2e_s = max_over_ranks(max(f0.elapsed_time(f1) / 1e3, 0.0))
        e2e = {"value": global_batch * steps / e2e_s, "unit": "tokens/s",
               "h2d_bytes_per_step": int(layers * U * (qpk + 2) * D * 4),
               "d2h_bytes_per_step": int(layers * U * qpk * D * 4),
               "steps": steps, "wall_s": wall, "l_timed": [l0 + warmup + 1, l0 + warmup + steps],
               "path": "kivi_decode_layers_host (C-ABI, one call per step over all layers, "
                       "pinned host buffers, copies in the timed region, returns with the "
                       "step's outputs on the host)",
               "step_graph": dict(kb.step_graph_stats(local),
                                  mode=os.environ.get("KIVI_STEP_GRAPH", "auto (single-layer steps)"))}
        seq_used = [(hk[j % pool, 0].numpy(), hv[j % pool, 0].numpy(), hq[j % pool, 0].numpy())
                    for j in range(warmup + steps)]
        last_out = ho[0].numpy().copy()
    else:
        seq_used = [(ks[j % pool, 0].cpu().numpy(), vs[j % pool, 0].cpu().numpy(),
                     qs[j % pool, 0].cpu().numpy()) for j in range(warmup + steps)]
        last_out = outs[0].cpu().numpy()

    # ---- optional NCCL all-gather of every layer's outputs ------
    gather = None
    if args.gather:
        from paper_2402_02750_b200.sharding import gather_outputs, partition_units
        batch = CONFIGS[args.config][2]
        counts = [U] * world if scaling == "weak" else \
            [len(partition_units(batch, heads, world, r)) for r in range(world)]
        for ly in range(layers):
            gather_outputs(outs[ly], counts)
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(steps):
            for ly in range(layers):
                gather_outputs(outs[ly], counts)
        g1.record(stream)
        barrier()
        g_s = max_over_ranks(g0.elapsed_time(g1) / 1e3)
        gbytes = layers * sum(counts) * qpk * D * 4
        gather = {"ms_per_step": g_s / steps * 1e3, "bytes_per_step": gbytes,
                  "GBps": gbytes * steps / g_s / 1e9 if g_s > 0 else None,
                  "collective": "all_gather_into_tensor (NCCL)" if world > 1 else "none (1 rank)",
                  "note": "timed separately; not part of value"}

    # ---- reference legs (rank 0, N = 1): CPU baseline + sampled-unit parity ---
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            rate, sample, kind, _, _ = cpu_reference_sample(
                args.config, steps=min(8, steps), warmup=1, threads=threads,
                units=32 * threads, bits=bits)
            step_s = layers * heads * (global_batch // world) * qpk / rate
            cpu = {"value": (global_batch // world) / step_s, "unit": "tokens/s",
                   "cores": threads, "kind": kind, "sample": sample}
        except Exception as e:  # the checker is optional for our own arm
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
        if do_parity and prompts:
            try:
                torch.cuda.synchronize()
                states = {u: caches[0].export_unit(u) for u in prompts}
                outs_u = {u: last_out[u] for u in prompts}
                parity = reference_parity_sample(bits, qpk, prompts, seq_used, outs_u, states)
            except Exception as e:
                parity = {"error": str(e)}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            ent = tj.get("configs", {}).get(f"{args.config}/{bits}")
            if ent:
                traffic = ent.get("dram_bytes_per_launch")
        except Exception:
            pass

    if rank == 0:
        config["l_timed"] = [l0 + warmup + 1, l0 + warmup + steps]
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": data_note(args),
            "config": config,
            "l2": l2_note,
            "hbm_gbs_per_gpu_step": alg_bytes / elapsed / 1e9,
            "step_latency_ms": latency,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_spec_8TBs": achieved / 8000.0,
                         "kernel": attend_kernel_name(qpk, U, ctx),
                         "bytes_per_launch": per_launch_bytes, "avg_launch_us": avg_launch_s * 1e6,
                         "kernel_share_of_step": avg_launch_s * layers / (elapsed / steps),
                         "launches_timed": kern_n,
                         "timing": "separate pass (same l window): CUDA events around every "
                                   "attend launch; the `value` pass records none"},
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": launches,
            "gather": gather,
            "clocks": clocks.summary(),
            "remeasured": remeasured,
        }
        print(json.dumps(line), flush=True)
    for c in caches:
        c.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=0, help="override layer count (debug)")
    ap.add_argument("--bits", type=int, default=0, choices=[0, 2, 4],
                    help="override the config's bit width (C4 sweeps 2 and 4)")
    ap.add_argument("--data", choices=["normal", "uniform"], default="normal",
                    help="synthetic K/V/q distribution (SURVEY §8d: N(0, 1))")
    ap.add_argument("--outliers", action="store_true",
                    help="key channels {1, 17, 40} x 50 (the reference's outlier analysis)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--gather", action="store_true",
                    help="also time the optional NCCL all-gather of every layer's outputs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: batch per GPU (default); strong: fixed global batch (c4, c5)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU rehearsal of the rank/launch path (gloo, no GPU work)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    if args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
