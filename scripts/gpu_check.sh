# Quick check of the working tree on the B200: smoke, GPU suite, chosen bench lines,
# K2 DRAM bytes on C5 (the traffic figure of the bench roofline).
# usage: TAG=r04a CONFIGS="c7 c5" bash scripts/gpu_check.sh
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_${TAG}.log
if [ -z "$NOTESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests_${TAG}.log
fi
for c in ${CONFIGS:-c7 c5}; do
  st=10; case $c in c1|c2a|c2) st=50;; esac
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --compare off > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
  grep '^{' gpurun_out/bench_${c}_${TAG}.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], 'ms', round(d['ms_per_step'],4), 'frac', round(r['frac'],4), r.get('smem_frac_executed'), 'parity', str(d.get('parity'))[:80])"
done
if [ -n "$NCU_C5" ]; then
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k2_tiled -s 1 -c 1 \
    python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --graph off --compare off > gpurun_out/ncu_c5_dram_${TAG}.txt 2>&1; echo ncu_c5=$?
grep -E 'dram__|gpu__time' gpurun_out/ncu_c5_dram_${TAG}.txt
fi
echo done
