# K6 build-flag A/B: bench configs for each PQTOPK_NVCC_EXTRA variant in $FLAGSETS (";"-separated)
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mean %.4f median %.4f ms'%(d['ms_per_step'], d['step_ms']['median']), 'frac %.3f'%d['roofline']['frac'], d['parity'][:36])"; }
IFS=';' read -ra SETS <<< "${FLAGSETS:-;-DK6_NO_GTH_CODE}"
i=0
for F in "${SETS[@]}"; do
  PQTOPK_NVCC_EXTRA="$F" python -m paper_2408_09992_b200.build --force > gpurun_out/build_f$i.log 2>&1; echo "build [$F] rc=$?"
  for c in ${CONFIGS:-c7 c2a}; do
    for v in ${VARIANTS:-legacy}; do
      ex=""; [ $v = legacy ] && ex="--tuning users_per_row=16"
      timeout 600 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 $ex > gpurun_out/bench_${c}_${v}_f$i.log 2>&1
      echo "[$F] $c $v $(summ gpurun_out/bench_${c}_${v}_f$i.log)"
    done
  done
  i=$((i+1))
done
