# K2 v3 shrink-watermark A/B (PQTOPK_K2_WMIN) on the batched configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step %.4f k2 %.4f frac %.3f'%(d['step_ms']['median'], d['roofline']['per_launch']['k2_ms'], d['roofline']['frac']), d['parity'][:24])" 2>/dev/null || tail -2 $1; }
for c in ${CONFIGS:-c2 c3 c4}; do
  for w in ${WMS:-0 256 1024 4096}; do
    st=20; [ $c = c4 ] && st=5; [ $c = c5 ] && st=3
    PQTOPK_K2_WMIN=$w timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/bench_${c}_wm${w}.log 2>&1
    echo "$c wm>=$w $(summ gpurun_out/bench_${c}_wm${w}.log)"
  done
done
