# usage: CFG=c3 TAG=v2b bash scripts/prof_k2.sh
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_ -s 3 -c 1 -o gpurun_out/k2_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_full_${CFG}_${TAG}.log
