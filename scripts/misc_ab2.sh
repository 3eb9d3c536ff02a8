python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "layout or tiled or paired" > gpurun_out/gputests_lay.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gputests_lay.log)"
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], 'create %.2f'%d['create_s'])" 2>&1 | tail -1; }
for c in c6 c2; do for v in gpu host; do env=""; [ $v = host ] && env="PQTOPK_HOST_LAYOUT=1"
  env $env timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_lay$v.log 2>&1; echo "$c layout=$v $(summ gpurun_out/bench_${c}_lay$v.log)"; done; done
for c in c1 c2a; do for ch in 0 1 2 4 8 37 74; do tun=""; [ $ch != 0 ] && tun="--tuning chunks=$ch"
  timeout 600 python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline $tun > gpurun_out/bench_${c}_ch$ch.log 2>&1; echo "$c chunks=$ch $(summ gpurun_out/bench_${c}_ch$ch.log)"; done; done
