# C2 knob sweep on the final build (same box)
cd "$(dirname "$0")/.." && TAG=${1:-swb}
run() { env "$@" timeout 300 python bench.py --config c2 --steps 32 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/sw.json 2>/dev/null; python3 -c "import json;j=json.load(open('gpurun_out/sw.json'));r=j['roofline'];print('$*', round(j['value']), round(r['avg_launch_us'],1), 'us', round(r['frac'],3), j['clocks']['sm_mhz'])"; }
for rep in 1 2; do
run KIVI_TAIL_CTAS=1
run KIVI_TAIL_CTAS=2
run KIVI_VIMMA=0
run KIVI_TAIL_SUB=128
run KIVI_BODY_SUB=512
done
