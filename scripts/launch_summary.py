"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum launch list."""
import collections, csv, sys
rows = list(csv.reader([l for l in open(sys.argv[1]) if l.startswith('"')]))
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.Counter(), collections.Counter()
for r in data:
    name = r[ik]
    for key in ("attend_body", "attend_tail", "combine", "append_fast", "append_kernel", "prefill",
                "uniform", "normalize", "attend_generic", "materialize"):
        if key in name:
            name = key
            break
    else:
        name = name[:48]
    tot[name] += float(r[iv].replace(",", "")); cnt[name] += 1
for k, v in tot.most_common():
    print(f"{k:48s} n={cnt[k]:5d} total_us={v/1000:10.1f} avg_us={v/cnt[k]/1000:8.2f}")
