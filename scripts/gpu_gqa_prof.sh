# GQA (C3) evidence: launch list + one full ncu capture of the GQA attend kernel; e2e diagnostics.
cd "$(dirname "$0")/.." && TAG=${1:-gqa}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv python bench.py --config c3 --layers 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c3_$TAG.log 2>&1; echo NCU_LAUNCH $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_gqa" -s 6 -c 1 -o gpurun_out/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo NCU_FULL $?
timeout 600 python scripts/e2e_diag.py > gpurun_out/e2e_diag_$TAG.log 2>&1; echo E2E $?; cat gpurun_out/e2e_diag_$TAG.log
