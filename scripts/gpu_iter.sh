# usage: bash scripts/gpu_iter.sh TAG — parity (fast path + state), bench (no cpu baseline), launch list, ncu of body/tail
cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $? ; tail -2 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 8 > /dev/null 2>&1; echo NCU_LAUNCH $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_(body|tail)" -s 10 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 6 > gpurun_out/ncu_$TAG.log 2>&1; echo NCU $?
