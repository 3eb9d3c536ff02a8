# K6 round-size / candidate-buffer A/B (compile-time) on c7 and the K6 small shapes
mkdir -p gpurun_out
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('median %.4f ms'%d['step_ms']['median'], 'frac %.3f'%d['roofline']['frac'])" 2>/dev/null || tail -2 $1; }
for v in "16384 0" "16384 512" "24576 512" "32768 512"; do
  set -- $v
  PQTOPK_NVCC_EXTRA="-DK6_STAGE_BYTES=$1 -DK6_CAP_SLACK=$2" python -m paper_2408_09992_b200.build --force > gpurun_out/build_st$1_$2.log 2>&1 || { echo "build $v failed"; tail -3 gpurun_out/build_st$1_$2.log; continue; }
  timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "fused" > gpurun_out/t_st$1_$2.log 2>&1; echo "stage $1 slack $2 tests: $(tail -1 gpurun_out/t_st$1_$2.log)"
  for c in c7 c2a; do
    ex=""; [ $c = c2a ] && ex="--tuning variant=5"
    timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline $ex > gpurun_out/b_${c}_st$1_$2.log 2>&1
    echo "  $c $(summ gpurun_out/b_${c}_st$1_$2.log)"
  done
done
python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
