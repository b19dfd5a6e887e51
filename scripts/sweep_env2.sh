# usage: bash scripts/sweep_env2.sh CONFIG "VAR1=a VAR2=b" "VAR1=c ..." ... — attend us/launch per env set
cd "$(dirname "$0")/.." && CFG=$1 && shift
for e in "$@"; do
  env $e timeout 300 python bench.py --config $CFG --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep.json 2>/dev/null
  python3 -c "import json;j=json.load(open('gpurun_out/sweep.json'));r=j['roofline'];print('$e', round(r['avg_launch_us'],1), 'us', round(r['frac'],3))"
done
