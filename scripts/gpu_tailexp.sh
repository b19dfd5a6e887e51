cd "$(dirname "$0")/.."
for cfg in "0 1" "1 2" "1 3" "1 2" "0 1" "1 3"; do set -- $cfg
  KIVI_TAIL_SIDE=$1 KIVI_TAIL_CTAS=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 64 > gpurun_out/tailexp_$1_$2.json 2>/dev/null
  python3 -c "import json;j=json.load(open('gpurun_out/tailexp_$1_$2.json'));r=j['roofline'];print('side=$1 ctas=$2', round(j['value']), round(r['avg_launch_us'],1), round(r['frac'],3), j['clocks']['sm_mhz'], j['clocks']['reasons'])"
done
