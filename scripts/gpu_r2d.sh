# usage: bash scripts/gpu_r2d.sh TAG — full gpu tests (no -x), smoke, e2e probe, facade acceptance, C2 launch list
cd "$(dirname "$0")/.." && TAG=${1:-x}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu -rf -s -k "facade" > gpurun_out/pytest_facade_$TAG.log 2>&1; echo PYTEST_FACADE $?; grep -E "^\[|passed|failed" gpurun_out/pytest_facade_$TAG.log | tail -14
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -8 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo SMOKE $?; tail -2 gpurun_out/smoke_$TAG.log
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe_$TAG.txt 2>&1; echo PROBE $?; cat gpurun_out/e2e_probe_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo NCU_LAUNCH $?
python scripts/launch_summary.py gpurun_out/launches_c2_$TAG.csv > gpurun_out/launches_c2_${TAG}_summary.txt 2>&1; head -30 gpurun_out/launches_c2_${TAG}_summary.txt
