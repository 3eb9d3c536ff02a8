# K2 time and DRAM bytes of one config against K2 launch tunings.
# usage: CFG=c5 TUS="none ctas=128 ctas=128,chunks=15" TAG=x bash scripts/tuning_ab.sh
mkdir -p gpurun_out
TAG=${TAG:-tu}
for tun in ${TUS:-none}; do
  tu=""; [ "$tun" != none ] && tu="--tuning $tun"
  nm=$(echo $tun | tr ',=' '__')
  timeout 600 python bench.py --config ${CFG:-c5} --steps ${STEPS:-5} --warmup 3 --compare off --no-cpu-baseline $tu > gpurun_out/${TAG}_${nm}.log 2>&1; echo bench_$nm=$?
  grep '^{' gpurun_out/${TAG}_${nm}.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$tun', 'ms', round(d['ms_per_step'],4), 'k2', round(r['per_launch']['k2_ms'],4), 'frac', round(r['frac'],4), 'frac_exec', r.get('smem_frac_executed'))"
  [ -n "$NONCU" ] && continue
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k2_tiled -s 1 -c 1 \
    python bench.py --config ${CFG:-c5} --steps 1 --warmup 1 --no-cpu-baseline --graph off --compare off $tu > gpurun_out/${TAG}_ncu_${nm}.txt 2>&1
  grep -E 'dram__|gpu__time' gpurun_out/${TAG}_ncu_${nm}.txt
done
