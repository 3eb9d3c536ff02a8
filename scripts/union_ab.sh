# Union floors A/B (PQTOPK_K2_UNION=0 turns them off): GPU suite, then per config
# the bench line and K2's DRAM bytes with and without.
mkdir -p gpurun_out
TAG=${TAG:-un}
if [ -z "$NOTESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests_${TAG}.log
fi
for c in ${CONFIGS:-c5 c3}; do
 for un in 1 0; do
  st=5; [ $c = c2 ] && st=50
  PQTOPK_K2_UNION=$un timeout 600 python bench.py --config $c --steps $st --warmup 3 --compare off --no-cpu-baseline > gpurun_out/${TAG}_${c}_u$un.log 2>&1; echo bench_${c}_u$un=$?
  grep '^{' gpurun_out/${TAG}_${c}_u$un.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c union=$un', 'ms', round(d['ms_per_step'],4), 'k2', round(r['per_launch']['k2_ms'],4), 'frac', round(r['frac'],4), 'exec', r.get('smem_frac_executed'), 'parity', str(d.get('parity'))[:70])"
  [ -n "$NONCU" ] && continue
  PQTOPK_K2_UNION=$un timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k2_tiled -s 1 -c 1 \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --graph off --compare off > gpurun_out/${TAG}_ncu_${c}_u$un.txt 2>&1
  grep -E 'dram__|gpu__time' gpurun_out/${TAG}_ncu_${c}_u$un.txt
 done
done
