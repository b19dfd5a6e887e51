# prefill kernel times (ncu launch list) of the in-tree library and variants in vtmp/
cd "$(dirname "$0")/.." && cp paper_2402_02750_b200/libkivi_b200.so /tmp/base.so
for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so; else cp vtmp/$v.so paper_2402_02750_b200/libkivi_b200.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prefill --csv --log-file gpurun_out/pf_$v.csv python bench.py --layers 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
  python3 - $v <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(f"gpurun_out/pf_{sys.argv[1]}.csv")) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]: d[r[ki].split('(')[0].split('::')[-1]].append(float(r[vi])/1000)
print(sys.argv[1], {k:(len(v), round(sum(v)/len(v),1)) for k,v in d.items()})
PY
done
cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so
