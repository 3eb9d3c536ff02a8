# ncu --set full of one K6 launch (config $C, tuning via PQTOPK_TUNING env: e.g. users_per_row=16)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in ${VARIANTS:-px legacy}; do
  tun=""; [ $v = legacy ] && tun="users_per_row=16"
  PQTOPK_TUNING=$tun timeout 900 ncu --set full --clock-control none --import-source on -k regex:k6_query -s 3 -c 1 \
     -o gpurun_out/k6_${C:-c7}_${v}_${TAG:-x} python scripts/trace_k6_run.py ${C:-c7} /dev/null > gpurun_out/ncu_k6_${v}.log 2>&1
  echo "$v rc=$?"
  python scripts/ncu_summary.py gpurun_out/k6_${C:-c7}_${v}_${TAG:-x}.ncu-rep > gpurun_out/k6_${C:-c7}_${v}_${TAG:-x}_summary.txt 2>&1
  cat gpurun_out/k6_${C:-c7}_${v}_${TAG:-x}_summary.txt
done
