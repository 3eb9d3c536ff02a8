# ncu --set full (with SASS source) of one K7 launch + the stall hot spots
mkdir -p gpurun_out
TAG=${TAG:-k7}; C=${C:-c2a}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_resident -s 3 -c 1 \
   -o gpurun_out/k7_${C}_${TAG} python scripts/trace_k6_run.py $C /dev/null > gpurun_out/ncu_k7_${TAG}.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/k7_${C}_${TAG}.ncu-rep
python scripts/ncu_src_regions.py gpurun_out/k7_${C}_${TAG}.ncu-rep 6
