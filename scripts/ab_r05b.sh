mkdir -p gpurun_out
PQTOPK_NVCC_EXTRA="-DK2_TRACE" python -m paper_2408_09992_b200.build --force > gpurun_out/r05_build_trace.log 2>&1; echo "trace build rc=$?"
for c in c2 c3; do
for v in "4 1" "1 0"; do
  set -- $v
  PQTOPK_K2_SEEDDIV=$1 PQTOPK_K2_FIRST_SHRINK=$2 PQTOPK_K2_DEBUG=1 timeout 300 python scripts/trace_k2_run.py $c gpurun_out/r05_k2_${c}_s$1_f$2.trace > gpurun_out/r05_trace_run_${c}_s$1_f$2.log 2>&1; echo "trace run $c $v rc=$?"
  grep "k2_tiled debug" gpurun_out/r05_trace_run_${c}_s$1_f$2.log | tail -3
  python scripts/trace_k2.py gpurun_out/r05_k2_${c}_s$1_f$2.trace 6 1 2>&1 | tail -14
done
done
