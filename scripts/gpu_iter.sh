# usage: bash gpu_iter.sh TAG  — fast-path parity, bench (no cpu baseline), ncu of the fast kernel
cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fast or single or passthrough" > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $? ; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_(body|tail)" -s 6 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_$TAG.log 2>&1; echo NCU $?
