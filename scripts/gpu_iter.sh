# Iteration check: build, K2 parity subset (or all with ALL=1), bench configs, optional ncu of k2_tiled.
# usage: TAG=v3b CONFIGS="c4 c3" PROF="c4" ALL=1 bash scripts/gpu_iter.sh
mkdir -p gpurun_out
TAG=${TAG:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
SEL=${TESTSEL:-"tiled or paired or random or geometry or invariants"}
if [ -n "$ALL" ]; then SEL=""; fi
timeout 900 python -m pytest tests -m gpu -q --timeout 300 ${SEL:+-k "$SEL"} > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_${TAG}.log | tail -12
for c in ${CONFIGS:-c4 c3 c2}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
  python - <<PY
import json
l=[x for x in open('gpurun_out/bench_${c}_${TAG}.log') if x.startswith('{')]
if not l: print(open('gpurun_out/bench_${c}_${TAG}.log').read()[-1500:])
else:
    d=json.loads(l[-1]); r=d['roofline']
    print('${c}', d['config']['k2_plan'], 'ms/step %.3f'%d['ms_per_step'], 'k2 %.3f ms'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], d['clocks']['sm_mhz'])
PY
done
for c in ${PROF}; do
CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline ${BENCHARGS}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k2_tiled} -s 3 -c 1 -o gpurun_out/k2_${c}_${TAG} $CMD > gpurun_out/ncu_full_${c}_${TAG}.log 2>&1; echo ncu_$c=$?
done
