mkdir -p gpurun_out
TAG=${TAG:-v3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "tiled" > gpurun_out/gpu_tiled_${TAG}.log 2>&1; echo tiled=$?
tail -30 gpurun_out/gpu_tiled_${TAG}.log | grep -E "passed|failed|Error|assert" | head -20
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED" gpurun_out/gpu_tests_${TAG}.log | tail -12
for c in ${CONFIGS:-c4 c3 c2}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
  python - <<PY
import json
l=[x for x in open('gpurun_out/bench_${c}_${TAG}.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_${c}_${TAG}.log').read()[-1500:])
else:
    d=json.loads(l[-1]); r=d['roofline']
    print('${c}', d['config']['k2_plan'], 'ms/step %.2f'%d['ms_per_step'], 'k2 %.2f ms'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], d['clocks']['sm_mhz'])
PY
done
