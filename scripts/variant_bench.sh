# usage: bash scripts/variant_bench.sh CONFIG [variant ...] — attend us/launch of the in-tree library
# ("base") and each variants/NAME.so swapped in, all on this box
cd "$(dirname "$0")/.." && CFG=$1 && shift
cp paper_2402_02750_b200/libkivi_b200.so /tmp/base.so
for v in base "$@" base "$@"; do
  if [ "$v" = base ]; then cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so; else cp $( [ -f variants/$v.so ] && echo variants || echo vtmp )/$v.so paper_2402_02750_b200/libkivi_b200.so; fi
  timeout 300 python bench.py --config $CFG --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vb.json 2>gpurun_out/vb.err || tail -3 gpurun_out/vb.err
  python3 -c "import json;j=json.load(open('gpurun_out/vb.json'));r=j['roofline'];print('$v', round(r['avg_launch_us'],1), 'us', round(r['frac'],3), 'value', round(j['value']), j['clocks']['sm_mhz'])"
done
cp /tmp/base.so paper_2402_02750_b200/libkivi_b200.so
