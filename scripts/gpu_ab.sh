# usage: bash scripts/gpu_ab.sh TAG ENVVAR "v1 v2" [configs] — parity tests then A/B bench of an env knob
cd "$(dirname "$0")/.." && TAG=$1; VAR=$2; VALS=$3; CFGS=${4:-c2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -m gpu -x > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -4 gpurun_out/pytest_$TAG.log
for c in $CFGS; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_${c}_$v.json 2> gpurun_out/bench_${TAG}_${c}_$v.err
  python - "$c" "$v" gpurun_out/bench_${TAG}_${c}_$v.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1]); r=d["roofline"]
    print(f"{sys.argv[1]} {sys.argv[2]}: value {d['value']:.1f} tok/s  attend {r['avg_launch_us']:.1f} us  frac {r['frac']:.3f}  sm {d['clocks']['sm_mhz']}  parity {d.get('parity') and d['parity'].get('max_rel_l2')}")
except Exception as e: print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
done; done
