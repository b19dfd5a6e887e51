cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -q -m gpu -x -k "gqa or GQA or c3 or C3 or qpk or decode_layers or mha_tc or MHA_TC" > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c3_$TAG.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c3', round(d['value'],1), round(r['avg_launch_us'],1), round(r['frac'],3), d['clocks']['sm_mhz'])"
bash scripts/gpu_c3prof.sh $TAG 2>&1 | grep -E "time_duration|issue_active|bank_conflicts|stalls"
