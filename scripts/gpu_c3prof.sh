cd "$(dirname "$0")/.." && TAG=${1:-c3p}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_gqa_tc" -s 3 -c 1 -o gpurun_out/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo NCU_C3 $?
python scripts/ncu_summary.py gpurun_out/prof_c3_$TAG.ncu-rep 10 > gpurun_out/ncu_c3_${TAG}_summary.txt 2>&1; head -24 gpurun_out/ncu_c3_${TAG}_summary.txt
