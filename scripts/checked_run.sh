# Memory-safety / hang evidence without compute-sanitizer (closed on this GPU pool):
#  1. the checked build (libpqtopk_checked.so, -DPQTOPK_CHECKED: device-side bounds
#     checks on code loads, shared-table offsets, candidate buffers and merge scratch,
#     bounded spin-waits / mbarrier waits that trap with the failing site);
#  2. every kernel family (scripts/sanitize_cases.py) under it, REPS times each
#     (each run is an oracle parity check, so a race shows up as a parity failure);
#  3. the whole GPU parity suite under the checked build.
# usage (on the GPU box): TAG=r02c bash scripts/checked_run.sh
mkdir -p gpurun_out/checked
TAG=${TAG:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/checked/build.log 2>&1; echo build=$?
python -m paper_2408_09992_b200.build --checked >> gpurun_out/checked/build.log 2>&1; echo build_checked=$?
for c in ${CASES:-tiled16 tiled8 tiled4 tiledbal latency k6grid k6clus k6pair k7 k7clus merge subset recjpq dense}; do
  log=gpurun_out/checked/case_${c}_${TAG}.log
  PQTOPK_CHECKED=1 timeout ${TLIM:-600} python scripts/sanitize_cases.py --reps ${REPS:-20} $c > $log 2>&1
  rc=$?
  echo "checked $c rc=$rc $(grep -cE '^ok ' $log) ok-runs $(grep -E 'PQ_DCHECK|PARITY FAIL|Error' $log | head -2 | tr '\n' ' ')" | tee -a gpurun_out/checked/summary_${TAG}.txt
done
PQTOPK_CHECKED=1 timeout ${TLIM2:-1500} python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/checked/gputests_checked_${TAG}.log 2>&1
echo "checked gpu suite rc=$? $(tail -1 gpurun_out/checked/gputests_checked_${TAG}.log)" | tee -a gpurun_out/checked/summary_${TAG}.txt
grep -c PQ_DCHECK gpurun_out/checked/*_${TAG}.log | tee -a gpurun_out/checked/summary_${TAG}.txt
