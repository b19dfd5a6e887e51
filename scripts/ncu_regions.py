"""Per-region stall breakdown of one kernel's ncu source page.
usage: ncu_regions.py SOURCE_CSV [BUCKET_BYTES]   (SOURCE_CSV from
  ncu -i REP --page source --csv --print-source sass -k regex:NAME)"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
bucket = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x400
hdr = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
if "--" in sys.argv: pass
ia, isrc = hdr.index("Address"), hdr.index("Source")
isamp, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
sc = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
tot = sum(int(r[isamp] or 0) for r in data)
reg = collections.OrderedDict()
for r in data:
    off = int(r[ia], 16) - base
    b = off // bucket * bucket
    e = reg.setdefault(b, [0, 0, collections.Counter(), collections.Counter()])
    s = int(r[isamp] or 0)
    e[0] += s
    e[1] += int(r[iex] or 0)
    op = r[isrc].split()[0] if not r[isrc].strip().startswith("@") else r[isrc].split()[1]
    e[3][op.split(".")[0]] += int(r[iex] or 0)
    for i, n in sc:
        e[2][n] += int(r[i] or 0)
for b, (s, n, st, ops) in reg.items():
    if s < tot * 0.01:
        continue
    print(f"{b:#07x} samples {100*s/tot:5.1f}%  inst {n:>10d}  stalls: " +
          ", ".join(f"{k}={100*v/max(s,1):.0f}%" for k, v in st.most_common(5)) +
          "  ops: " + ", ".join(f"{k}:{v}" for k, v in ops.most_common(6)))
