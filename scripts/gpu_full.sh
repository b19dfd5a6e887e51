# Full round evidence: tests, smoke, bench (ours + reference arm), ncu launch list + full capture.
cd "$(dirname "$0")/.." && TAG=${1:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep "Model name" >> gpurun_out/gpu_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo SMOKE $?; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>&1; echo REF $?; cat gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo NCU_LAUNCH $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_(body|tail)" -s 10 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 6 > gpurun_out/ncu_$TAG.log 2>&1; echo NCU_FULL $?
# exercise the multi-rank code path (torchrun, NCCL) with the 1 GPU available
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 16 --warmup 3 --no-cpu-baseline --gather > gpurun_out/torchrun_$TAG.json 2> gpurun_out/torchrun_$TAG.err; echo TORCHRUN $?; cat gpurun_out/torchrun_$TAG.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 4 --warmup 3 > gpurun_out/torchrun_ref_$TAG.json 2>&1; echo TORCHRUN_REF $?; tail -1 gpurun_out/torchrun_ref_$TAG.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_gqa_tc" -s 3 -c 1 -o gpurun_out/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo NCU_C3 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv python bench.py --config c3 --layers 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo NCU_LAUNCH_C3 $?
