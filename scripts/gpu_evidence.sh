# Round evidence: build, smoke, full GPU tests, default bench (with cpu_baseline), reference arm,
# ncu launch list of the bench command, ncu --set full of the dominant kernel.
# usage: TAG=r01v3 bash scripts/gpu_evidence.sh
mkdir -p gpurun_out
TAG=${TAG:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed" gpurun_out/gpu_tests_${TAG}.log | tail -3
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_default_${TAG}.log | tail -1 | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu_launch=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_c4_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu_full=$?
