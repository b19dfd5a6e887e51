# e2e with and without the per-step CUDA graph (KIVI_STEP_GRAPH) on C1 / C2
cd "$(dirname "$0")/.." && TAG=${1:-g}
for c in ${CFGS:-c1 c2}; do for v in 0 1 0 1; do
  KIVI_STEP_GRAPH=$v timeout 600 python bench.py --config $c --steps 64 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/gr_${TAG}_${c}_$v.json 2>/dev/null
  python -c "
import json; j=json.load(open('gpurun_out/gr_${TAG}_${c}_$v.json')); e=j['e2e']
print('$c graph=$v value', round(j['value']), 'e2e', round(e['value']), e['step_graph'], j['clocks']['sm_mhz'])"
done; done
