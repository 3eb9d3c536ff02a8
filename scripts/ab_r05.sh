# C2/C3 per-unit fixed costs: seeding fraction / first-tile shrink knobs, then a K2 trace with the unit timeline.
mkdir -p gpurun_out
summ() { grep "^{" $1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('ms %.4f'%d['ms_per_step'], 'median %.4f'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.4f'%r['frac'], (d.get('parity') or '')[:40])" 2>&1 | tail -1; }
for v in "4 1" "2 1" "1 1" "1 0" "2 0" "8 1"; do
  set -- $v
  for c in c2 c3; do
    st=10; [ $c = c2 ] && st=50
    PQTOPK_K2_SEEDDIV=$1 PQTOPK_K2_FIRST_SHRINK=$2 timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/r05_${c}_s$1_f$2.log 2>&1; echo "seeddiv $1 first_shrink $2 $c $(summ gpurun_out/r05_${c}_s$1_f$2.log)"
  done
done
PQTOPK_NVCC_EXTRA="-DK2_TRACE" python -m paper_2408_09992_b200.build --force > gpurun_out/r05_build_trace.log 2>&1; echo "trace build rc=$?"
for v in "4 1" "1 0"; do
  set -- $v
  PQTOPK_K2_SEEDDIV=$1 PQTOPK_K2_FIRST_SHRINK=$2 PQTOPK_K2_DEBUG=1 timeout 300 python scripts/trace_k2_run.py c2 gpurun_out/r05_k2_c2_s$1_f$2.trace > gpurun_out/r05_trace_run_c2_s$1_f$2.log 2>&1; echo "trace run rc=$?"
  grep "k2_tiled debug" gpurun_out/r05_trace_run_c2_s$1_f$2.log | tail -3
  python scripts/trace_k2.py gpurun_out/r05_k2_c2_s$1_f$2.trace 6 1 2>&1 | tail -14
done
