cd "$(dirname "$0")/.." && TAG=${1:-qp}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"append_flush|prefill_values|prefill_keys" -c 4 -o gpurun_out/prof_$TAG python bench.py --layers 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/ncu_$TAG.log 2>&1; echo NCU $?
python scripts/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep 8 > gpurun_out/ncu_${TAG}_summary.txt 2>&1; cat gpurun_out/ncu_${TAG}_summary.txt | head -120
