# A/B two versions of k2_tiled.cu on the same box (write scripts/ab/k2_tiled_A.cu and _B.cu first, e.g. from git show):
# usage: CFG=c4 TUNINGS=warps=16 bash scripts/ab/ab.sh   (prints "A|B k2 <ms> frac <f>" twice each)
rm -f gpurun_out/sweep_results.txt
for v in A B A B; do
  cp scripts/ab/k2_tiled_$v.cu paper_2408_09992_b200/csrc/k2_tiled.cu
  python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
  CFG=${CFG:-c4} TUNINGS="${TUNINGS:-chunks=37}" bash scripts/sweep.sh > /dev/null 2>&1
  echo "$v $(tail -1 gpurun_out/sweep_results.txt | grep -o 'k2 [0-9.]* ms frac [0-9.]*')"
done
