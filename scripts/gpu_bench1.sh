set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep "Model name"
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo BENCH_EXIT $?
tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 300 python bench.py --impl reference --steps 8 --warmup 3 > gpurun_out/bench_ref1.json 2>&1; echo REF_EXIT $?
cat gpurun_out/bench_ref1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.json 2>&1; echo NCU1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attend_fast -s 3 -c 1 -o gpurun_out/prof_fast1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_full.log 2>&1; echo NCU2 $?
tail -5 gpurun_out/ncu_full.log
