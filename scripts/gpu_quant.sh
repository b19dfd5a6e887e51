# Quantizer kernels: full GPU suite + per-kernel times of prefill / append / flush.
cd "$(dirname "$0")/.." && TAG=${1:-q}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --layers 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1; echo NCU $?
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv
python - gpurun_out/launches_$TAG.csv <<'PY'
import csv,collections,sys
rows=list(csv.reader([l for l in open(sys.argv[1]) if l.startswith('"')]))
hdr=rows[0]; ik=hdr.index("Kernel Name"); iv=hdr.index("Metric Value")
tot=collections.Counter(); cnt=collections.Counter()
for r in rows[1:]:
    n=r[ik]
    if 'prefill' in n or 'flush' in n:
        n=n.split('(')[0][-44:]; tot[n]+=float(r[iv].replace(',',''));cnt[n]+=1
for k,v in tot.items(): print(' ',k,cnt[k],round(v/cnt[k]/1000,1),'us')
PY
