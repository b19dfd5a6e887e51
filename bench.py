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


PROF_STRIDE = 4   # time every 4th attend launch of each cache (bench loop below)


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


def cpu_reference_sample(cfg_name, steps, warmup, threads, units=None, bits=0):
    """Times the REFERENCE decode_attention (oracle/_ref, compiled from the
    reference sources) on a bounded sample of the workload's units; returns
    (unit-steps per second, description, kind)."""
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
            f"{threads} threads; extrapolated to {layers * heads * batch * qpk} unit-steps/step")
    return rate, desc, "reference"


def run_reference_arm(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    layers, heads, batch, ctx, bits, qpk, desc = CONFIGS[args.config]
    if args.bits:
        bits = args.bits
        desc = desc.replace("2-bit", f"{bits}-bit")
    threads = os.cpu_count() or 1
    # each "step" is a bounded sample: ~16 units per thread, one decode each
    rate, sample, kind = cpu_reference_sample(args.config, args.steps, args.warmup, threads,
                                              units=16 * threads, bits=bits)
    unit_steps_per_step = layers * heads * batch * qpk
    step_s = unit_steps_per_step / rate
    tok_s = batch / step_s
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32/f64 (reference CPU)", "data": "synthetic",
        "config": {"workload": desc, "layers": layers, "kv_heads": heads, "batch": batch,
                   "ctx": ctx, "bits": bits, "group_size": G, "residual": R, "head_dim": D,
                   "q_per_kv": qpk},
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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

    layers, heads, batch, ctx, bits, qpk, desc = CONFIGS[args.config]
    if args.layers:
        layers = args.layers
    if args.bits:
        bits = args.bits
        desc = desc.replace("2-bit", f"{bits}-bit")
    from paper_2402_02750_b200.sharding import partition_units
    scaling = args.scaling or ("strong" if args.config in ("c4", "c5") else "weak")
    capacity_note = None
    if scaling == "strong":
        # fixed global batch, units partitioned over ranks (no collective)
        U = len(partition_units(batch, heads, world, rank))
        global_batch = batch
    else:
        # every rank serves its own batch (data-parallel replicas)
        U = batch * heads
        global_batch = batch * world
    steps, warmup = args.steps, args.warmup
    # C4 (Llama-2-13B, batch 256: 2-bit ~287 GB, 4-bit ~344 GB of state) does
    # not fit one 180 GB B200 (SURVEY §7 hard part 5).  When a rank's share
    # does not fit, it runs the largest power-of-two batch that does, and the
    # line says so; at 8 GPUs (32 sequences per GPU) the full job fits.
    free, _ = torch.cuda.mem_get_info(dev)
    per_unit = state_bytes_per_unit(ctx + steps + warmup + R, bits, layers) + 2 * 4 * D * ctx
    if U * per_unit > 0.85 * free:
        b_rank = max(1, U // heads)
        while b_rank > 1 and b_rank * heads * per_unit > 0.85 * free:
            b_rank //= 2
        capacity_note = (f"{U // heads} sequences/GPU need {U * per_unit / 1e9:.0f} GB of "
                         f"state > {free / 1e9:.0f} GB free: timed {b_rank} sequences/GPU")
        U = b_rank * heads
        global_batch = b_rank * world
        scaling = "weak"
    l0 = ctx - warmup - steps
    if l0 < 1:
        raise SystemExit("--steps + --warmup must be < ctx")
    cfg = kb.CacheConfig(bits, G, R, D)

    # ---- build the state: prefill every layer on the device ----------------
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    caches = []
    kbuf = torch.empty((U, l0, D), device=dev, dtype=torch.float32)
    vbuf = torch.empty_like(kbuf)
    for _ in range(layers):
        c = kb.KVCache(cfg, U, capacity_tokens=ctx + steps + warmup + R, device=local)
        kbuf.uniform_(-1.0, 1.0, generator=gen)
        vbuf.uniform_(-1.0, 1.0, generator=gen)
        c.prefill(kbuf, vbuf)
        c.set_attend_path("auto")
        caches.append(c)
    del kbuf, vbuf
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    # per-step inputs resident in HBM (a pool of 2 sets per layer, cycled)
    pool = 2
    qs = torch.empty((pool, layers, U, qpk, D), device=dev).uniform_(-1, 1, generator=gen)
    ks = torch.empty((pool, layers, U, D), device=dev).uniform_(-1, 1, generator=gen)
    vs = torch.empty((pool, layers, U, D), device=dev).uniform_(-1, 1, generator=gen)
    outs = torch.empty((layers, U, qpk, D), device=dev)

    def step(i):
        p = i % pool
        for ly in range(layers):
            caches[ly].decode(qs[p, ly], ks[p, ly], vs[p, ly], q_per_kv=qpk, out=outs[ly])

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

    for i in range(warmup):
        step(i)
    barrier()
    # the attend kernel's launch time (roofline) comes from CUDA events the
    # library records around it inside the timed region, on every
    # PROF_STRIDE-th launch of each cache: the events cost host time, which
    # latency-bound steps (C1: 38 vs 44 us/step with every launch timed)
    # would otherwise pay in `value`
    prof = 0 if os.environ.get("KIVI_BENCH_NOPROF") else PROF_STRIDE
    for c in caches:
        c.profile_read()
        c.profile_enable(prof)
    l_start = caches[0].total_tokens
    # ---- timed region (device-resident inputs) ------------------------------
    # A state smaller than 4x L2 (C1: 18.6 MB vs 126 MB) would be served from
    # L2: then every timed step is bracketed by its own events and L2 is
    # flushed (a 2x-L2 write) between steps, outside the events.
    stream = torch.cuda.current_stream()
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    state_total = U * state_bytes_per_unit(ctx + steps + warmup + R, bits, layers)
    flush = state_total < 4 * l2
    scratch = torch.empty((2 * l2) // 4, dtype=torch.float32, device=dev) if flush else None
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        if flush:
            evs = []
            for i in range(steps):
                scratch.fill_(float(i))
                a_ = torch.cuda.Event(enable_timing=True)
                b_ = torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                step(warmup + i)
                b_.record(stream)
                evs.append((a_, b_))
        else:
            e0.record(stream)
            for i in range(steps):
                step(warmup + i)
            e1.record(stream)
        barrier()
    if flush:
        elapsed = max_over_ranks(sum(a_.elapsed_time(b_) for a_, b_ in evs) / 1e3)
    else:
        elapsed = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    l2_note = (f"state {state_total / 1e6:.1f} MB < 4x L2 ({l2 >> 20} MB): L2 flushed by a "
               f"{2 * l2 >> 20} MB write between timed steps (per-step events)" if flush else
               f"state {state_total / 1e9:.1f} GB >> {l2 >> 20} MB L2 (inputs larger than L2, "
               "no flush)")
    kern_ms, kern_n, launches = 0.0, 0, 0
    for c in caches:
        ms, n, tot = c.profile_read()
        kern_ms += ms
        kern_n += n   # launches timed
        launches += tot
        c.profile_enable(False)

    # algorithmic bytes of the timed attends (l after each append), per launch
    alg_bytes = sum(attend_bytes_per_unit(l_start + i + 1, bits, qpk) for i in range(steps))
    alg_bytes *= U * layers
    per_launch_bytes = alg_bytes / (steps * layers)
    avg_launch_s = (kern_ms / 1e3) / max(kern_n, 1)
    achieved = per_launch_bytes / avg_launch_s / 1e9 if avg_launch_s > 0 else float("nan")
    peak, peak_src = load_peaks()

    tok_s = global_batch * steps / elapsed
    ms_per_step = elapsed / steps * 1e3

    # ---- e2e through the C-ABI host-buffer entry point ------------------------
    e2e = None
    if not args.no_e2e:
        hq = torch.empty((pool, layers, U, qpk, D), dtype=torch.float32, pin_memory=True)
        hk = torch.empty((pool, layers, U, D), dtype=torch.float32, pin_memory=True)
        hv = torch.empty((pool, layers, U, D), dtype=torch.float32, pin_memory=True)
        ho = torch.empty((layers, U, qpk, D), dtype=torch.float32, pin_memory=True)
        hq.copy_(qs.cpu())
        hk.copy_(ks.cpu())
        hv.copy_(vs.cpu())
        # same workload, continuing the decode: l runs past ctx.  W untimed
        # steps first, as for the device-resident loop: a cache's first host
        # call creates its staging buffers, copy stream and events (one-time,
        # ~40 ms per cache).
        e2e_steps = steps
        for i in range(warmup):
            for ly in range(layers):
                caches[ly].decode_host(hq[i % pool, ly], hk[i % pool, ly], hv[i % pool, ly],
                                       ho[ly], q_per_kv=qpk)
        barrier()
        t0 = time.perf_counter()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        dbg = os.environ.get("KIVI_E2E_DEBUG")
        for i in range(e2e_steps):
            p = i % pool
            tw = time.perf_counter()
            for ly in range(layers):
                caches[ly].decode_host(hq[p, ly], hk[p, ly], hv[p, ly], ho[ly], q_per_kv=qpk)
            for c in caches:  # this step's outputs are on the host before the next
                c.host_join(stream)
            if dbg:
                te = time.perf_counter() - tw
                torch.cuda.synchronize()
                print(f"e2e step {i}: enqueue {te * 1e3:.2f} ms, wall {(time.perf_counter() - tw) * 1e3:.2f} ms",
                      file=sys.stderr, flush=True)
        f1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
        e2e_s = max_over_ranks(max(f0.elapsed_time(f1) / 1e3, 0.0))
        e2e = {"value": global_batch * e2e_steps / e2e_s, "unit": "tokens/s",
               "h2d_bytes_per_step": int(layers * U * (qpk + 2) * D * 4),
               "d2h_bytes_per_step": int(layers * U * qpk * D * 4),
               "steps": e2e_steps, "wall_s": wall,
               "path": "kivi_decode_host (C-ABI, pinned host buffers, copies in the timed region)"}

    # ---- optional NCCL all-gather of every layer's outputs ------
    gather = None
    if args.gather:
        from paper_2402_02750_b200.sharding import gather_outputs
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            rate, sample, kind = cpu_reference_sample(args.config, steps=min(8, steps),
                                                      warmup=1, threads=threads,
                                                      units=32 * threads, bits=bits)
            step_s = layers * heads * batch * qpk / rate
            cpu = {"value": batch / step_s, "unit": "tokens/s", "cores": threads, "kind": kind,
                   "sample": sample}
        except Exception as e:  # the checker is optional for our own arm
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            if tj.get("config") == args.config and tj.get("bits") == bits:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass

    if rank == 0:
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (uniform(-1,1) K/V/q generated on device)",
            "config": {"workload": desc, "name": args.config, "layers": layers,
                       "kv_heads": heads, "batch_per_gpu": global_batch / world,
                       "global_batch": global_batch,
                       "ctx": ctx, "bits": bits, "group_size": G, "residual": R, "head_dim": D,
                       "q_per_kv": qpk, "units_per_layer_per_gpu": U,
                       "capacity_limited": capacity_note,
                       "l_timed": [l_start + 1, l_start + steps],
                       "l2": l2_note,
                       "parallelism": f"dp{world} ({scaling}; units sharded by "
                                      "(batch, kv-head), no collective)"},
            "hbm_gbs_per_gpu_step": alg_bytes / elapsed / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "frac_of_spec_8TBs": achieved / 8000.0,
                         "kernel": attend_kernel_name(qpk, U, ctx),
                         "bytes_per_launch": per_launch_bytes, "avg_launch_us": avg_launch_s * 1e6,
                         "kernel_share_of_step": avg_launch_s * steps * layers / elapsed,
                         "launches_timed": kern_n},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gather": gather,
            "clocks": clocks.summary(),
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
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", action="store_true",
                    help="also time the optional NCCL all-gather of every layer's outputs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: batch per GPU (default); strong: fixed global batch (c4, c5)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
