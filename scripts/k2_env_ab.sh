# K2 v3 env-toggle A/B: bench per config for "def" and each variable in $ENVS (VAR=VALUE, space-separated)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], (d['parity'] or '')[:30])" 2>&1 | tail -1; }
if [ -n "$TESTSEL" ]; then for e in $ENVS; do env $e timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_env.log 2>&1; echo "[$e] tests rc=$? $(tail -1 gpurun_out/gputests_env.log)"; done; fi
for c in ${CONFIGS:-c2 c3 c4 c5}; do
  for e in def $ENVS; do
    ee=""; [ $e != def ] && ee=$e
    env $ee timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 ${BENCHARGS:---no-cpu-baseline} > gpurun_out/bench_${c}_env.log 2>&1
    echo "$c [$e] $(summ gpurun_out/bench_${c}_env.log)"
  done
done
