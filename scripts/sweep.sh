# usage: CFG=c4 TUNINGS="warps=8 warps=16,chunks=18" bash scripts/sweep.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for t in ${TUNINGS}; do
  timeout 600 python bench.py --config ${CFG:-c4} --steps 3 --warmup 3 --no-cpu-baseline --tuning "$t" > gpurun_out/sweep.log 2>&1
  python - <<PY
import json
l=[x for x in open('gpurun_out/sweep.log') if x.startswith('{')]
if not l: print(open('gpurun_out/sweep.log').read()[-800:])
else:
    d=json.loads(l[-1]); r=d['roofline']
    msg = " ".join(["${CFG:-c4}", "$t", str(d["config"]["k2_plan"]), "k2 %.3f ms" % r["per_launch"]["k2_ms"], "frac %.3f" % r["frac"]])
    print(msg); open("gpurun_out/sweep_results.txt", "a").write(msg + "\n")
PY
done
