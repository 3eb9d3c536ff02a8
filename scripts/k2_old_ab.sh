# current vs round-1 tree (_old_r01/) bench lines, same box
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], (d['parity'] or '')[:44])" 2>&1 | tail -1; }
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo build=$?
(cd _old_r01 && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo oldbuild=$?)
if [ -n "$TESTSEL" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_oldab.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gputests_oldab.log)"; fi
for c in ${CONFIGS:-c2 c3 c4 c5 c6}; do
  for v in new old; do
    dir=.; [ $v = old ] && dir=_old_r01
    (cd $dir && timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > $OLDPWD/gpurun_out/bench_${c}_${v}_ab.log 2>&1)
    echo "$c $v $(summ gpurun_out/bench_${c}_${v}_ab.log)"
  done
done
