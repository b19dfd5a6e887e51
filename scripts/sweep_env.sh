# usage: bash scripts/sweep_env.sh CONFIG VAR v1 v2 ... — attend us/launch per env value (no e2e/cpu)
cd "$(dirname "$0")/.." && CFG=$1 && VAR=$2 && shift 2
for v in "$@"; do
  env $VAR=$v timeout 300 python bench.py --config $CFG --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep.json 2>/dev/null
  python3 -c "import json;j=json.load(open('gpurun_out/sweep.json'));r=j['roofline'];print('$VAR=$v', round(r['avg_launch_us'],1), 'us', round(r['frac'],3))"
done
