cd "$(dirname "$0")/.." && TAG=${1:-x}
timeout 300 python scripts/proj_split_probe.py > gpurun_out/proj_split_$TAG.txt 2>&1; echo PROBE $?; cat gpurun_out/proj_split_$TAG.txt | tail -12
timeout 300 python scripts/driver_probe.py 2>&1 | tail -12
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/driver_probe.py 2>&1 | tail -12
