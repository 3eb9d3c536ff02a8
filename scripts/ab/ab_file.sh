# A/B two versions of one csrc file on the same box:
#   FILE=k6_query.cu CFGS="c1 c2a c7" ARGS="--tuning cluster=8" bash scripts/ab/ab_file.sh
# expects scripts/ab/A_<FILE> and scripts/ab/B_<FILE>; prints "<v> <cfg> us/step k2_us frac"
F=${FILE:-k6_query.cu}
for v in A B A B; do
  cp scripts/ab/${v}_$F paper_2408_09992_b200/csrc/$F
  python -m paper_2408_09992_b200.build --force > /dev/null 2>&1
  for c in ${CFGS:-c1 c2a}; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $ARGS 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v', '$c', round(d['ms_per_step']*1e3,1), 'us/step', round(r['per_launch']['k2_ms']*1e3,1), 'us k', round(r['frac'],3))"
  done
done
