# ncu --set full of one K2 v3 launch per config (source-level), summary + per-line stalls
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${CONFIGS:-c2}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_tiled -s 2 -c 1 \
     -o gpurun_out/k2_${c}_${TAG:-x} python scripts/trace_k2_run.py $c /dev/null > gpurun_out/ncu_k2_${c}.log 2>&1
  echo "$c rc=$?"
  python scripts/ncu_summary.py gpurun_out/k2_${c}_${TAG:-x}.ncu-rep > gpurun_out/k2_${c}_${TAG:-x}_summary.txt 2>&1
  cat gpurun_out/k2_${c}_${TAG:-x}_summary.txt
  python scripts/ncu_lines.py gpurun_out/k2_${c}_${TAG:-x}.ncu-rep 30 > gpurun_out/k2_${c}_${TAG:-x}_lines.txt 2>&1
  cat gpurun_out/k2_${c}_${TAG:-x}_lines.txt
done
