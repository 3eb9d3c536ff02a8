mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo bench=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -30; tail -3 gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench_c4.log
