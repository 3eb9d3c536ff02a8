# Evidence pass (rounds 3+): build, smoke, full GPU tests, default bench line (C4 with
# cpu_baseline), every config's bench line, one-rank NCCL path, reference arm,
# ncu launch lists, ncu --set full of the dominant kernel per path.
# usage: TAG=r03g bash scripts/gpu_evidence_r03.sh
mkdir -p gpurun_out
TAG=${TAG:-ev3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_${TAG}.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
tail -1 gpurun_out/gpu_tests_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_default_${TAG}.log | tail -1 | cut -c1-220
for c in ${CONFIGS:-c1 c2a c2 c3 c5 c6 c7 c7b}; do
  st=10; case $c in c1|c2a|c2) st=50;; esac
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 \
    bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bench_c4_torchrun1_${TAG}.log 2>&1; echo bench_torchrun1=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref=$?
# launch lists (the same commands as the bench lines, graph off so every launch is listed)
for c in c4 c2 c2a c1; do
  n=400; [ $c = c4 ] && n=60
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c $n --csv --log-file gpurun_out/launches_${c}_${TAG}.csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --graph off --compare off > /dev/null 2>&1; echo ncu_launch_$c=$?
done
# full captures of the dominant kernel
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_c4_${TAG} \
    python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --graph off --compare off > /dev/null 2>&1; echo ncu_c4=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_c2_${TAG} \
    python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --graph off --compare off > /dev/null 2>&1; echo ncu_c2=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_c5_${TAG} \
    python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --graph off --compare off > /dev/null 2>&1; echo ncu_c5=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k6_query -s 3 -c 1 -o gpurun_out/k6_c7_${TAG} \
    python scripts/trace_k6_run.py c7 /dev/null > /dev/null 2>&1; echo ncu_c7=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_resident -s 3 -c 1 -o gpurun_out/k7_c2a_${TAG} \
    python scripts/trace_k6_run.py c2a /dev/null > /dev/null 2>&1; echo ncu_c2a=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_resident -s 3 -c 1 -o gpurun_out/k7_c1_${TAG} \
    python scripts/trace_k6_run.py c1 /dev/null > /dev/null 2>&1; echo ncu_c1=$?
for r in k2_c4 k2_c2 k2_c5 k6_c7 k7_c2a k7_c1; do
  python scripts/ncu_summary.py gpurun_out/${r}_${TAG}.ncu-rep > gpurun_out/${r}_${TAG}_ncu.txt 2>&1
done
rm -f gpurun_out/*_${TAG}.ncu-rep   # (summarised above; gpurun brings back at most 64 MiB)
for c in c4 c2 c2a c1; do python scripts/launch_list.py gpurun_out/launches_${c}_${TAG}.csv > gpurun_out/launches_${c}_${TAG}_summary.txt 2>&1; done
echo done
