# Round evidence: build, smoke, full GPU tests, default bench line (C4, with cpu_baseline),
# every config's bench line, reference arm, ncu launch list, ncu --set full of the dominant kernel.
# usage: TAG=r01f bash scripts/gpu_evidence.sh
mkdir -p gpurun_out
TAG=${TAG:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo tests=$?
grep -E "passed|failed" gpurun_out/gpu_tests_${TAG}.log | tail -3
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; echo bench=$?
grep '^{' gpurun_out/bench_default_${TAG}.log | tail -1 | cut -c1-200
for c in ${CONFIGS:-c1 c2a c2 c3 c5 c6 c7 c7b}; do
  st=10; case $c in c1|c2a|c2) st=50;; esac
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/bench_${c}_${TAG}.log 2>&1; echo bench_$c=$?
done
# the sharded (NCCL all-gather + packed merge) path, one rank on this one-GPU box
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 \
    bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/bench_c4_torchrun1_${TAG}.log 2>&1; echo bench_torchrun1=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.log 2>&1; echo ref=$?
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --graph off"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo ncu_launch=$?
for c in ${PROFCFG:-c4 c5}; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_${c}_${TAG} python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --graph off > gpurun_out/ncu_full_${c}_${TAG}.log 2>&1; echo ncu_full_$c=$?
done
# the fused small-batch kernel (K6): launch list and one full capture on the B = 1 configs
for c in ${K6CFG:-c2a c1}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${c}_${TAG}.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --graph off > /dev/null 2>&1; echo ncu_launch_$c=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k6_query -s 3 -c 1 -o gpurun_out/k6_${c}_${TAG} python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --graph off > gpurun_out/ncu_full_k6_${c}_${TAG}.log 2>&1; echo ncu_full_k6_$c=$?
done
