python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c3 c4; do for ub in 4 8 16 32; do PQTOPK_K1_UB=$ub python scripts/k1_time.py $c; done; done
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1; }
for c in c2 c6 c4; do for v in gpu host; do env=""; [ $v = host ] && env="PQTOPK_HOST_LAYOUT=1"
  env $env timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_lay$v.log 2>&1; echo "$c layout=$v $(summ gpurun_out/bench_${c}_lay$v.log)"; done; done
