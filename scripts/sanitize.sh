# compute-sanitizer memcheck / racecheck / synccheck (+ initcheck) over every kernel family
# (scripts/sanitize_cases.py; each case is also an oracle parity check).
# usage (on the GPU box): TAG=r02a bash scripts/sanitize.sh
mkdir -p gpurun_out/sanitize
TAG=${TAG:-san}
CS=/usr/local/cuda/bin/compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sanitize/build.log 2>&1; echo build=$?
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in ${CASES:-tiled16 tiled8 tiled4 latency k6grid k6clus merge subset recjpq dense}; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    log=gpurun_out/sanitize/${tool}_${c}_${TAG}.log
    timeout ${TLIM:-900} $CS --tool $tool $extra --error-exitcode 17 --print-limit 50 \
        python scripts/sanitize_cases.py $c > $log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|PARITY FAIL|^ok " $log | tr '\n' ' ')
    echo "$tool $c rc=$rc $summ" | tee -a gpurun_out/sanitize/summary_${TAG}.txt
  done
done
