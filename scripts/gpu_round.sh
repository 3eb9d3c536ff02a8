mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -30; tail -2 gpurun_out/smoke.log
for c in ${CONFIGS:-c4 c2 c3}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo bench_$c=$?
  python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_$c.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_$c.log').read()[-2000:]); sys.exit()
d=json.loads(l[-1]); r=d['roofline']
print('$c', 'ms/step %.2f'%d['ms_per_step'], 'value %.3e'%d['value'], 'k2 %.2f ms'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], 'e2e %.3e'%d['e2e']['value'], d['parity'], d['clocks'])
"
done
