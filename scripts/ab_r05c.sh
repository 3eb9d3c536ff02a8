mkdir -p gpurun_out
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], d['config']['k2_plan']['ctas'], d['config']['k2_plan']['chunks'], (d.get('parity') or '')[:60])" 2>&1 | tail -1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "tiled or union or merge" > gpurun_out/r05c_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/r05c_tests.log)"
for bal in 0 1; do
  for c in ${CONFIGS:-c2 c3 c5}; do
    st=10; [ $c = c2 ] && st=50
    PQTOPK_K2_BAL=$bal timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/r05c_${c}_bal$bal.log 2>&1; echo "bal $bal $c $(summ gpurun_out/r05c_${c}_bal$bal.log)"
  done
done
for o in 4 8 16 24; do
  for c in c2 c3; do
    st=10; [ $c = c2 ] && st=50
    PQTOPK_K2_UNIT_OVH=$o timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/r05c_${c}_ovh$o.log 2>&1; echo "ovh $o $c $(summ gpurun_out/r05c_${c}_ovh$o.log)"
  done
done
