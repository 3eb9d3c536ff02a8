# K7 launch-attribute A/B (cooperative / PDL) on C1 and C2a
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
summ() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('median %.4f ms'%d['step_ms']['median'], 'warm %.4f'%d['step_ms'].get('warm_l2_median',0))" 2>/dev/null || tail -2 $1; }
for c in c1 c2a; do
  for v in def coop1 coop0 nopdl; do
    env=""
    [ $v = coop1 ] && env="PQTOPK_K7_COOP=1"
    [ $v = coop0 ] && env="PQTOPK_K7_COOP=0"
    [ $v = nopdl ] && env="PQTOPK_K7_NO_PDL=1"
    env $env timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${c}_${v}_la.log 2>&1
    echo "$c $v $(summ gpurun_out/bench_${c}_${v}_la.log)"
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c1_la.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --graph off > /dev/null 2>&1
python scripts/launch_list.py gpurun_out/launches_c1_la.csv 2>/dev/null | head -4
