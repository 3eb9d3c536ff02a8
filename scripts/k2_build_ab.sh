# K2 build-flag A/B: bench configs for each PQTOPK_NVCC_EXTRA variant in $FLAGSETS (";"-separated)
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('median %.4f ms'%d['step_ms']['median'], 'k2 %.4f'%r['per_launch']['k2_ms'], 'frac %.3f'%r['frac'], (d['parity'] or '')[:30])" 2>&1 | tail -1; }
IFS=';' read -ra SETS <<< "${FLAGSETS:-;-DK2_SLACK=2}"
i=0
for F in "${SETS[@]}"; do
  PQTOPK_NVCC_EXTRA="$F" python -m paper_2408_09992_b200.build --force > gpurun_out/build_k2f$i.log 2>&1; echo "build [$F] rc=$?"
  if [ -n "$TESTSEL" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "$TESTSEL" > gpurun_out/gputests_k2f$i.log 2>&1; echo "[$F] tests rc=$? $(tail -1 gpurun_out/gputests_k2f$i.log)"; fi
  for c in ${CONFIGS:-c5 c4 c3}; do
    st=${STEPS:-5}; [ $c = c2 ] && st=50; timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --compare off > gpurun_out/bench_${c}_k2f$i.log 2>&1
    echo "[$F] $c $(summ gpurun_out/bench_${c}_k2f$i.log)"
  done
  i=$((i+1))
done
