# K2 v3 A/B on the GPU box: bench lines per config and variant (env toggles).
# usage: TAG=r02j CONFIGS="c2 c3 c4" VARIANTS="def nopf" bash scripts/k2_ab.sh
mkdir -p gpurun_out
TAG=${TAG:-k2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo build=$?
if [ -n "$TESTSEL" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_${TAG}.log 2>&1; echo tests=$?; grep -E "passed|failed|FAILED|Error" gpurun_out/gputests_${TAG}.log | tail -5
fi
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('mean %.4f median %.4f ms'%(d['ms_per_step'], d['step_ms']['median']), 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], 'create %.2fs'%d['create_s'], (d['parity'] or '')[:40], d['config']['k2_plan'])" 2>&1 | tail -1; }
for c in ${CONFIGS:-c2 c3}; do
  for v in ${VARIANTS:-def nopf}; do
    env=""
    [ $v = nopf ] && env="PQTOPK_K2_NO_L2PF=1"
    [ $v = hostlayout ] && env="PQTOPK_HOST_LAYOUT=1"
    env $env timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 ${BENCHARGS} > gpurun_out/bench_${c}_${v}_${TAG}.log 2>&1
    echo "$c $v $(summ gpurun_out/bench_${c}_${v}_${TAG}.log)"
  done
done
