# ab_old (r03n library) vs HEAD build-flag variants, same box.  FLAGSETS=";-DK2_ASM_LDS"
mkdir -p gpurun_out
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], (d.get('parity') or '')[:40])" 2>&1 | tail -1; }
for c in ${CONFIGS:-c4 c3 c2}; do
  st=10; [ $c = c2 ] && st=50
  (cd ab_old && timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > ../gpurun_out/abb_old_${c}.log 2>&1); echo "old $c $(summ gpurun_out/abb_old_${c}.log)"
done
TESTSEL="${TESTSEL:-tiled}" STEPS=10 bash scripts/k2_build_ab.sh
python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
