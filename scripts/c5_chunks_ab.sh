# C5: K2 time and DRAM bytes against the item-chunk count (units = 128 groups x chunks).
# usage: CH="0 15 8" TAG=x bash scripts/c5_chunks_ab.sh   (0 = the planner's choice)
mkdir -p gpurun_out
TAG=${TAG:-c5ch}
for ch in ${CH:-0 15 8}; do
  tu=""; [ "$ch" != 0 ] && tu="--tuning chunks=$ch"
  timeout 600 python bench.py --config ${CFG:-c5} --steps 5 --warmup 3 --compare off --no-cpu-baseline $tu > gpurun_out/${TAG}_ch${ch}.log 2>&1; echo bench_ch$ch=$?
  grep '^{' gpurun_out/${TAG}_ch${ch}.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('chunks', '$ch', 'ms', round(d['ms_per_step'],3), 'k2', round(r['per_launch']['k2_ms'],3), 'frac_exec', r.get('smem_frac_executed'), 'parity', str(d.get('parity'))[:60])"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k2_tiled -s 1 -c 1 \
    python bench.py --config ${CFG:-c5} --steps 1 --warmup 1 --no-cpu-baseline --graph off --compare off $tu > gpurun_out/${TAG}_ncu_ch${ch}.txt 2>&1
  grep -E 'dram__|gpu__time' gpurun_out/${TAG}_ncu_ch${ch}.txt
done
