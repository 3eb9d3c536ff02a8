# K7 vs K6 on the GPU box: fused tests, bench lines, K7 phase traces.
# usage: TAG=k7a CONFIGS="c2a c1" TRACE="c2a c1" bash scripts/k7_ab.sh
mkdir -p gpurun_out
TAG=${TAG:-k7}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo build=$?
if [ -n "$TESTSEL" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_${TAG}.log 2>&1; echo tests=$?; grep -E "passed|failed|FAILED|Error" gpurun_out/gputests_${TAG}.log | tail -8
fi
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mean %.4f median %.4f warmL2 %.4f ms'%(d['ms_per_step'], d['step_ms']['median'], d['step_ms'].get('warm_l2_median',0)), 'frac %.3f'%d['roofline']['frac'], d['parity'], d['config']['k2_plan']['variant'])" 2>/dev/null || tail -3 $1; }
for c in ${CONFIGS:-c2a c1}; do
  for v in ${VARIANTS:-k7 k6}; do
    ex=""; md=0
    np=""
    [ $v = k6 ] && ex="--tuning variant=5"
    [ $v = k6np ] && ex="--tuning variant=5" && np=1
    [ $v = k7np ] && np=1
    case $v in k7m*) md=${v#k7m};; esac
    env ${np:+PQTOPK_NO_PAIRED=1} PQTOPK_K7_MODE=$md timeout 600 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline $ex > gpurun_out/bench_${c}_${v}_${TAG}.log 2>&1
    echo "$c $v $(summ gpurun_out/bench_${c}_${v}_${TAG}.log)"
  done
done
if [ -n "$TRACE" ]; then
  PQTOPK_NVCC_EXTRA=-DK6_TRACE python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
  for c in ${TRACE}; do
  for md in ${TMODES:-0}; do
    PQTOPK_K7_MODE=$md timeout 600 python scripts/trace_k6_run.py $c gpurun_out/k7_${c}_m${md}_${TAG}.trace > /dev/null 2>&1
    python scripts/trace_k7.py gpurun_out/k7_${c}_m${md}_${TAG}.trace > gpurun_out/trace_${c}_m${md}_${TAG}.txt 2>&1
    echo "== trace $c mode $md"; cat gpurun_out/trace_${c}_m${md}_${TAG}.txt
  done
  done
  python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
fi
