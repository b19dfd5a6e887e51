cd "$(dirname "$0")/.." && TAG=${1:-x}
for spin in 1 0; do KIVI_FACADE_SPIN=$spin timeout 600 oracle/_ref/facade_acceptance 2>&1 | grep -E "criterion 1|criterion 2|failed"; done
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/pytest_$TAG.log 2>&1; echo PYTEST $?; grep -E "passed|failed|^FAILED" gpurun_out/pytest_$TAG.log | tail -12
grep -B5 "Error" gpurun_out/pytest_$TAG.log | head -60
