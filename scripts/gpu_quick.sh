mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -8
CONFIGS="${CONFIGS:-c3 c4 c2}" bash scripts/diag.sh
