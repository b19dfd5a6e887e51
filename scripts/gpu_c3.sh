# usage: bash scripts/gpu_c3.sh TAG [ncu] — GQA parity tests + C3 bench (+ optional ncu capture of the GQA kernel)
cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gqa" > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $? ; tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --config c3 --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/c3_$TAG.json 2> gpurun_out/c3_$TAG.err; echo BENCH $?; tail -2 gpurun_out/c3_$TAG.err
python3 -c "import json;j=json.load(open('gpurun_out/c3_$TAG.json'));r=j['roofline'];print('c3', round(j['value']), 'tok/s', round(j['ms_per_step'],3), 'ms/step', round(r['achieved']), 'GB/s', round(r['frac'],3), 'us/launch', round(r['avg_launch_us'],1), 'e2e', round(j['e2e']['value']), j['clocks'])"
if [ "$2" = "ncu" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_gqa_tc" -s 3 -c 1 -o gpurun_out/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo NCU_FULL $?
fi
