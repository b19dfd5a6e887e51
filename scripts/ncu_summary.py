"""Summarise an ncu report, per kernel: key metrics, stall reasons, hottest SASS
classes (grouped by execution count).  usage: ncu_summary.py REPORT [N_CLASSES]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
ncls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print(f"== {d.get('Kernel Name', '?')}  grid {d.get('Grid Size', '')} block {d.get('Block Size', '')}")
    for k in KEYS:
        if k in d:
            print(f"  {k:62s} {d[k]:>16s} {units[hdr.index(k)]}")
    st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
          float(d[h]) for h in hdr
          if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")
          and d[h]}
    print("  stalls per issue: " + ", ".join(f"{k}={v:.2f}" for k, v in
                                            sorted(st.items(), key=lambda kv: -kv[1]) if v > 0.05))
    kid = d.get("ID")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", kid, "--launch-count", "1"] if False else
                         ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + d.get("Kernel Name", "").split("(")[0].split("<")[0].split()[-1]],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    hi = [i for i, r in enumerate(srows) if "Source" in r]
    if not hi:
        continue
    shdr = srows[hi[0]]
    data = srows[hi[0] + 1:]
    isrc = shdr.index("Source")
    iex = shdr.index("Instructions Executed")
    isamp = shdr.index("Warp Stall Sampling (All Samples)")
    cls = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
    for r in data:
        try:
            n = int(r[iex])
            s = int(r[isamp])
        except Exception:
            continue
        t = r[isrc].strip().split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
        c = cls[n]
        c[0] += 1
        c[1] += n
        c[2] += s
        c[3][op] += 1
    ts = sum(v[2] for v in cls.values()) or 1
    tn = sum(v[1] for v in cls.values()) or 1
    print(f"  total warp-inst {tn}")
    for n, (cnt, ni, s, ops) in sorted(cls.items(), key=lambda kv: -kv[1][2])[:ncls]:
        print(f"    exec {n:9d} #inst {cnt:5d} inst {ni / tn * 100:5.1f}% samples {s / ts * 100:5.1f}%"
              f"  {dict(ops.most_common(6))}")
