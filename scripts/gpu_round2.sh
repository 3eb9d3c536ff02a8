# Round-2 GPU pass: build, smoke, full GPU suite, insert counts, create times, bench lines.
# usage: TAG=r02m CONFIGS="c4 c5 c7b" bash scripts/gpu_round2.sh
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_${TAG}.log
if [ -z "$NOTESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED" gpurun_out/gpu_tests_${TAG}.log | tail -8
fi
for c in ${INSERTS:-}; do timeout 900 python scripts/k2_inserts.py $c > gpurun_out/inserts_${c}_${TAG}.log 2>&1; echo "inserts $c rc=$?"; cat gpurun_out/inserts_${c}_${TAG}.log | tail -3; done
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mean %.4f median %.4f ms'%(d['ms_per_step'], d['step_ms']['median']), 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], 'create %.2fs'%d['create_s'], (d['parity'] or '')[:60], 'e2e/value %.3f'%(d['e2e']['value']/d['value']))" 2>&1 | tail -1; }
for c in ${CONFIGS:-c4}; do
  timeout 1500 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_${c}_${TAG}.log 2>&1
  echo "bench $c rc=$? $(summ gpurun_out/bench_${c}_${TAG}.log)"
done
