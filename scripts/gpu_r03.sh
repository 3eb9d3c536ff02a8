# Round-3 check on the GPU box: build, full GPU suite, short bench lines.
# usage: TAG=r03a CONFIGS="c2 c4 c7" bash scripts/gpu_r03.sh
mkdir -p gpurun_out
TAG=${TAG:-r03}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo build=$?
if [ -z "$NOTESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
tail -2 gpurun_out/gpu_tests_${TAG}.log
fi
for c in ${CONFIGS:-c2 c4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
  python - <<PY
import json
l=[x for x in open('gpurun_out/bench_${c}_${TAG}.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_${c}_${TAG}.log').read()[-1500:])
else:
    d=json.loads(l[-1]); r=d['roofline']
    print('${c}', 'variant', d['config']['k2_plan']['variant'], 'ms/step %.4f median %.4f'%(d['ms_per_step'], d['step_ms']['median']), 'k2 %.4f ms'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], 'e2e %.3g'%d['e2e']['value'], d['clocks']['sm_mhz'])
PY
done
