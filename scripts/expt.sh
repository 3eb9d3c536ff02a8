python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in ${CONFIGS:-c4}; do for e in ${EXPTS:-0 1 2 4 7}; do
PQTOPK_K2_EXPT=$e timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/expt.log 2>&1
python - <<PY
import json
l=[x for x in open('gpurun_out/expt.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
msg = "$c expt=$e " + ("k2 %.3f ms frac %.3f" % (d['roofline']['per_launch']['k2_ms'], d['roofline']['frac']) if d else open('gpurun_out/expt.log').read()[-300:])
print(msg); open('gpurun_out/expt_results.txt','a').write(msg+"\n")
PY
done; done
