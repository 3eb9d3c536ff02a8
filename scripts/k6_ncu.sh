# ncu --set full (with SASS source) of one K6 launch + the stall hot spots
mkdir -p gpurun_out
TAG=${TAG:-k6}; C=${C:-c7}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k6_query -s 3 -c 1 \
   -o gpurun_out/k6_${C}_${TAG} python scripts/trace_k6_run.py $C /dev/null > gpurun_out/ncu_k6_${TAG}.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/k6_${C}_${TAG}.ncu-rep
python scripts/ncu_src_regions.py gpurun_out/k6_${C}_${TAG}.ncu-rep ${MINS:-200}
