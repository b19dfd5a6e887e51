# All BASELINE configs on one GPU (C4 as its 2-bit vs 4-bit sweep), short runs, no CPU baseline.
cd "$(dirname "$0")/.."
run() {
  tag=$1; shift
  timeout 900 python bench.py "$@" --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$tag.json 2> gpurun_out/cfg_$tag.err
  echo "$tag rc=$?"; tail -2 gpurun_out/cfg_$tag.err
  python3 -c "import json;j=json.load(open('gpurun_out/cfg_$tag.json'));r=j['roofline'];c=j['config'];print('$tag', round(j['value']), 'tok/s', round(j['ms_per_step'],3), 'ms/step', round(r['achieved']), 'GB/s', round(r['frac'],3), 'us/launch', round(r['avg_launch_us'],1), 'e2e', round(j['e2e']['value']), 'batch/gpu', c['batch_per_gpu'], c.get('capacity_limited'), j['clocks']['sm_mhz'])"
}
run c1 --config c1
run c3 --config c3
run c4b2 --config c4 --bits 2
run c4b4 --config c4 --bits 4
run c5 --config c5
