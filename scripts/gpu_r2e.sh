cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 300 python scripts/proj_split_probe.py > gpurun_out/proj_split_$TAG.txt 2>&1; echo PROBE $?; cat gpurun_out/proj_split_$TAG.txt | tail -12
timeout 1200 python -m pytest tests -q -m gpu -rf -s -k "facade or native or zero_copy or run_decode or decode_layers" > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; grep -E "^\[|passed|failed|^FAILED|Error" gpurun_out/pytest_$TAG.log | tail -20
