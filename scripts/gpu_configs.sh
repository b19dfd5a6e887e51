cd "$(dirname "$0")/.."
for c in c1 c3 c5; do
  timeout 900 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/cfg_$c.err
  python3 -c "import json;j=json.load(open('gpurun_out/cfg_$c.json'));r=j['roofline'];print('$c', round(j['value']), 'tok/s', round(j['ms_per_step'],3), 'ms/step', round(r['achieved']), 'GB/s', round(r['frac'],3), 'e2e', round(j['e2e']['value']), j['clocks']['sm_mhz'])"
done
