# usage: bash scripts/gpu_prof.sh <config> <tag>
mkdir -p gpurun_out
CFG=${1:-c4}; TAG=${2:-v1}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launch_${CFG}_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_score -s 3 -c 1 -o gpurun_out/k2_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo rc=$?
tail -3 gpurun_out/plain_${CFG}_${TAG}.log | cut -c1-300; tail -5 gpurun_out/ncu_full_${CFG}_${TAG}.log
