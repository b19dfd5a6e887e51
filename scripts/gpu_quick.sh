# usage: bash scripts/gpu_quick.sh TAG "pytest -k expr" [bench args...] — selected gpu tests + one bench
cd "$(dirname "$0")/.." && TAG=${1:-x}; K=${2:-}; shift 2
timeout 900 python -m pytest tests -q -m gpu -x ${K:+-k "$K"} > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -12 gpurun_out/pytest_$TAG.log
if [ $# -gt 0 ]; then timeout 600 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; fi
