mkdir -p gpurun_out
TAG=${TAG:-v3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for c in ${CONFIGS:-c4 c3}; do
CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 3 -c 1 -o gpurun_out/k2_${c}_${TAG} $CMD > gpurun_out/ncu_full_${c}_${TAG}.log 2>&1; echo ncu_$c=$?
tail -2 gpurun_out/ncu_full_${c}_${TAG}.log
done
