# Round evidence at HEAD: tests, smoke, C2 bench + reference arm, ncu launch lists and
# full captures (C2 body+tail, C3 both GQA kernels, C5 body+tail), torchrun, every config.
cd "$(dirname "$0")/.." && TAG=${1:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep "Model name" >> gpurun_out/gpu_$TAG.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; tail -2 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo SMOKE $?; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo BENCH $?; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2>&1; echo REF $?; tail -1 gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1; echo NCU_LAUNCH $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_(body|tail)" -s 10 -c 2 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --layers 6 > gpurun_out/ncu_$TAG.log 2>&1; echo NCU_FULL $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attend_gqa" -s 6 -c 2 -o gpurun_out/prof_c3_$TAG python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --layers 4 > gpurun_out/ncu_c3_$TAG.log 2>&1; echo NCU_C3 $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_$TAG.csv python bench.py --config c3 --layers 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > /dev/null 2>&1; echo NCU_LAUNCH_C3 $?
timeout 900 ncu --set full --clock-control none -k regex:"attend_(body|tail)" -s 10 -c 2 -o gpurun_out/prof_c5_$TAG python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --layers 6 > gpurun_out/ncu_c5_$TAG.log 2>&1; echo NCU_C5 $?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 16 --warmup 3 --no-cpu-baseline --gather > gpurun_out/torchrun_$TAG.json 2> gpurun_out/torchrun_$TAG.err; echo TORCHRUN $?; tail -c 400 gpurun_out/torchrun_$TAG.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 4 --warmup 3 > gpurun_out/torchrun_ref_$TAG.json 2>&1; echo TORCHRUN_REF $?
bash scripts/gpu_configs.sh
for f in gpurun_out/cfg_*.json; do case $f in *_r2*|*_final*) ;; *) cp $f ${f%.json}_$TAG.json;; esac; done
