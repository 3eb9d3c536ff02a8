mkdir -p gpurun_out
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], d['config']['k2_plan']['ctas'], d['config']['k2_plan']['chunks'], (d.get('parity') or '')[:60])" 2>&1 | tail -1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r05e_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/r05e_tests.log)"
for rep in 1 2; do
for c in ${CONFIGS:-c2 c3 c5 c4}; do
  st=10; [ $c = c2 ] && st=50
  (cd ab_old && timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > ../gpurun_out/r05e_old_${c}.log 2>&1); echo "old $c $(summ gpurun_out/r05e_old_${c}.log)"
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/r05e_new_${c}.log 2>&1; echo "new $c $(summ gpurun_out/r05e_new_${c}.log)"
done
done
PQTOPK_NVCC_EXTRA="-DK2_TRACE" python -m paper_2408_09992_b200.build --force > gpurun_out/r05_build_trace.log 2>&1; echo "trace build rc=$?"
for c in c2; do
  PQTOPK_K2_DEBUG=1 timeout 300 python scripts/trace_k2_run.py $c gpurun_out/r05e_k2_$c.trace > gpurun_out/r05e_trace_run_$c.log 2>&1; echo "trace run rc=$?"
  grep "k2_tiled debug" gpurun_out/r05e_trace_run_$c.log | tail -3
  python scripts/trace_k2.py gpurun_out/r05e_k2_$c.trace 4 1 2>&1 | tail -12
done
