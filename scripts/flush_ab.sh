cd $GRAFT_REPO_ROOT
cp paper_2402_02750_b200/libkivi_b200.so /tmp/base.so
for v in ${VARIANTS:-base flushold base flushold}; do
  if [ $v = base ]; then cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so; else cp vtmp/$v.so paper_2402_02750_b200/libkivi_b200.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:append_flush --csv --log-file gpurun_out/fl_$v.csv python bench.py --layers 4 --steps 40 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1
  python3 - $v <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(f"gpurun_out/fl_{sys.argv[1]}.csv")) if len(r)>5]
h=rows[0]; gi=h.index('Grid Size'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]: d[r[gi]].append(float(r[vi])/1000)
print(sys.argv[1], {k:(len(v), round(sum(v)/len(v),2)) for k,v in d.items()})
PY
  timeout 300 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --no-parity --no-e2e > gpurun_out/fb.json 2>/dev/null; python3 -c "import json;j=json.load(open('gpurun_out/fb.json'));print('$v', round(j['value']), j['step_latency_ms'], j['clocks']['sm_mhz'])"
done
cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so
[ -n "$NOTEST" ] || timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_random.py -q -x 2>&1 | tail -2
