# usage: bash scripts/gpu_r2b.sh TAG — full gpu tests, smoke, bench C2 (with cpu baseline), C1, C3
cd "$(dirname "$0")/.." && TAG=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo SMOKE $?; tail -3 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
for c in c1 c3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo BENCH_$c $?; tail -2 gpurun_out/bench_${c}_$TAG.err; cat gpurun_out/bench_${c}_$TAG.json; done
