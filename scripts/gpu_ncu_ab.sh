# usage: bash scripts/gpu_ncu_ab.sh TAG ENVVAR "v1 v2" KERNEL_REGEX [config] — ncu --set full of one kernel per variant
cd "$(dirname "$0")/.." && TAG=$1; VAR=$2; VALS=$3; KRE=$4; CFG=${5:-c2}
for v in $VALS; do
  env $VAR=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 6 -c 1 -o gpurun_out/prof_${TAG}_$v python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --layers 4 > gpurun_out/ncu_${TAG}_$v.log 2>&1; echo NCU_$v $?
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$v.ncu-rep 10 > gpurun_out/ncu_${TAG}_${v}_summary.txt 2>&1; head -40 gpurun_out/ncu_${TAG}_${v}_summary.txt
done
