# K2 v3 tile-end slack A/B: parity (tiled tests) + debug fractions + bench per slack
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], (d['parity'] or '')[:44])" 2>&1 | tail -1; }
for S in ${SLACKS:-1 2 3}; do
  export PQTOPK_K2_SLACK=$S
  if [ -n "$TESTSEL" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_slack$S.log 2>&1; echo "S=$S tests rc=$? $(tail -1 gpurun_out/gputests_slack$S.log)"; fi
  for c in ${CONFIGS:-c2 c3 c4 c5}; do
    timeout 600 python scripts/k2_inserts.py $c 2>&1 | grep "end-of-tile" | sed "s/^/S=$S $c /"
    timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 > gpurun_out/bench_${c}_slack$S.log 2>&1
    echo "S=$S $c $(summ gpurun_out/bench_${c}_slack$S.log)"
  done
done
