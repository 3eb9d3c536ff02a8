# same-box A/B of library variants living in directories ($DIRS, each a copy of the repo's runtime files with its own libpqtopk.so)
mkdir -p gpurun_out
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], d['config']['k2_plan']['ctas'], d['config']['k2_plan']['chunks'], (d.get('parity') or '')[:60])" 2>&1 | tail -1; }
for rep in 1 2; do
for c in ${CONFIGS:-c2 c3 c5}; do
  st=10; [ $c = c2 ] && st=50
  for d in ${DIRS:-ab_old ab_v1 ab_v2 .}; do
    n=$(echo $d | tr -d './'); n=${n:-cur}
    (cd $d && timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > $OLDPWD/gpurun_out/abd_${n}_${c}.log 2>&1); echo "$n $c $(summ gpurun_out/abd_${n}_${c}.log)"
  done
done
done
