# K7 diagnostics on the GPU box: phase traces cold / warm L2, one ncu --set full capture.
# usage: TAG=k7c C=c2a MODE=4 bash scripts/k7_diag.sh
mkdir -p gpurun_out
TAG=${TAG:-k7}; C=${C:-c2a}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export PQTOPK_K7_MODE=${MODE:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_resident -s 3 -c 1 \
   -o gpurun_out/k7_${C}_${TAG} python scripts/trace_k6_run.py $C /dev/null > gpurun_out/ncu_k7_${TAG}.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py gpurun_out/k7_${C}_${TAG}.ncu-rep > gpurun_out/k7_${C}_${TAG}_summary.txt 2>&1
cat gpurun_out/k7_${C}_${TAG}_summary.txt
PQTOPK_NVCC_EXTRA=-DK6_TRACE python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
for nf in 0 1; do
  TRACE_NOFLUSH=$nf timeout 600 python scripts/trace_k6_run.py $C gpurun_out/k7_${C}_nf${nf}_${TAG}.trace > /dev/null 2>&1
  echo "== trace $C noflush=$nf"; python scripts/trace_k7.py gpurun_out/k7_${C}_nf${nf}_${TAG}.trace
done
python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
