# Round-2 evidence at HEAD: full run (tests, smoke, bench, reference arm, ncu) + every config.
cd "$(dirname "$0")/.." && TAG=${1:-r2h}
bash scripts/gpu_full.sh $TAG
bash scripts/gpu_configs.sh
for f in gpurun_out/cfg_*.json; do cp $f ${f%.json}_$TAG.json; done
