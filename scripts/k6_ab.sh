# K6 A/B on the GPU box: tests, bench lines (variants below), phase traces.
# usage: TAG=r02f VARIANTS="def legacy legnogth old" TRACE="c7" bash scripts/k6_ab.sh
mkdir -p gpurun_out
TAG=${TAG:-k6}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo build=$?
if [ -d _old_r01 ]; then (cd _old_r01 && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1); fi
if [ -n "$TESTSEL" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_${TAG}.log 2>&1; echo tests=$?; grep -E "passed|failed|FAILED|Error" gpurun_out/gputests_${TAG}.log | tail -5
fi
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mean %.4f median %.4f ms'%(d['ms_per_step'], d['step_ms']['median']), 'frac %.3f'%d['roofline']['frac'], d['parity'][:40], d['config']['k2_plan'].get('prefix_splits'), d['config']['k2_plan'].get('table_copies'))"; }
for c in ${CONFIGS:-c2a c7 c1}; do
  for v in ${VARIANTS:-def legacy}; do
    ex=""; env=""; dir=.
    [ $v = legacy ] && ex="--tuning users_per_row=16"
    [ $v = legnogth ] && ex="--tuning users_per_row=16" && env="PQTOPK_K6_NO_GTH=1"
    [ $v = nogth ] && env="PQTOPK_K6_NO_GTH=1"
    [ $v = late ] && env="PQTOPK_K6_TMA_LATE=1"
    [ $v = old ] && dir=_old_r01
    (cd $dir && env $env timeout 600 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 $ex > $OLDPWD/gpurun_out/bench_${c}_${v}_${TAG}.log 2>&1)
    echo "$c $v $(summ gpurun_out/bench_${c}_${v}_${TAG}.log)"
  done
done
if [ -n "$TRACE" ]; then
  PQTOPK_NVCC_EXTRA=-DK6_TRACE python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
  for c in ${TRACE}; do
    timeout 600 python scripts/trace_k6_run.py $c gpurun_out/k6_${c}_${TAG}.trace > /dev/null 2>&1
    python scripts/trace_k6.py gpurun_out/k6_${c}_${TAG}.trace > gpurun_out/trace_${c}_${TAG}.txt 2>&1
    echo "== trace $c"; cat gpurun_out/trace_${c}_${TAG}.txt
  done
fi
