# Round-4 A/B pass: (1) r03n library (ab_old/) vs HEAD on the same box, (2) m = 64 on 32-user rows with
# 2-split phases (PQTOPK_K2_R32P=1) vs the paired 16-user layout, (3) C5 chunk counts vs DRAM bytes.
mkdir -p gpurun_out
TAG=${TAG:-ab4}
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], 'create %.2f'%d.get('create_s',-1), (d.get('parity') or '')[:40])" 2>&1 | tail -1; }
if [ -d ab_old ] && [ -z "$NOOLD" ]; then
for rep in 1 2; do
  for c in ${ABCFG:-c4 c3 c2}; do
    st=10; [ $c = c2 ] && st=50
    (cd ab_old && timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > ../gpurun_out/${TAG}_old_${c}_$rep.log 2>&1); echo "old $c rep$rep $(summ gpurun_out/${TAG}_old_${c}_$rep.log)"
    timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/${TAG}_new_${c}_$rep.log 2>&1; echo "new $c rep$rep $(summ gpurun_out/${TAG}_new_${c}_$rep.log)"
  done
done
fi
if [ -z "$NOC6" ]; then
PQTOPK_K2_R32P=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "tiled or geometry or boundaries" > gpurun_out/${TAG}_tests_r32p.log 2>&1; echo "tests r32p rc=$? $(tail -1 gpurun_out/${TAG}_tests_r32p.log)"
for v in 1 0; do
  PQTOPK_K2_R32P=$v timeout 900 python bench.py --config c6 --steps 10 --warmup 3 --no-cpu-baseline --compare off > gpurun_out/${TAG}_c6_r32p$v.log 2>&1; echo "c6 r32p=$v rc=$? $(summ gpurun_out/${TAG}_c6_r32p$v.log)"
done
fi
if [ -z "$NOC5" ]; then CH="${CH:-0 15 8}" TAG=${TAG}_c5ch bash scripts/c5_chunks_ab.sh; fi
echo done
