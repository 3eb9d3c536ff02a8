mkdir -p gpurun_out
for c in ${CONFIGS:-c3 c4}; do
for v in ${VARIANTS:-2}; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/diag_${c}_v$v.log 2>&1
python -c "
import json
l=[x for x in open('gpurun_out/diag_${c}_v$v.log') if x.startswith('{')]
if not l: print(open('gpurun_out/diag_${c}_v$v.log').read()[-1500:]); raise SystemExit
d=json.loads(l[-1])
print('$c v$v', d['config']['k2_plan'], 'k2 %.3f ms'%d['roofline']['per_launch']['k2_ms'], 'frac %.3f'%d['roofline']['frac'], d['clocks']['sm_mhz'])
"
done; done
