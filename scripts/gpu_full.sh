# Full round check: build, smoke, GPU tests, bench (c4 default + others), launch list + ncu full of K2.
# usage: TAG=v2 CONFIGS="c4 c2 c3 c5" bash scripts/gpu_full.sh
mkdir -p gpurun_out
TAG=${TAG:-v2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_${TAG}.log | tail -12
for c in ${CONFIGS:-c4}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
  grep '^{' gpurun_out/bench_${c}_${TAG}.log | tail -1 | cut -c1-600
done
if [ -n "$PROF" ]; then
  CMD="python bench.py --config ${PCFG:-c4} --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${PCFG:-c4}_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu_launch=$?
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o gpurun_out/k2_${PCFG:-c4}_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu_full=$?
  tail -3 gpurun_out/ncu_full_${TAG}.log
fi
