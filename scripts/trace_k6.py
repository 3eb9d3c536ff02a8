"""Summarise a PQTOPK_K6_TRACE dump: per-CTA globaltimer stamps of the fused
K6 kernel (0 start, 1 phi staged, 2 S share computed + broadcast, 3 cluster
barrier passed, 4 chunk scored, 5 chunk list published, 6 merge done (last
CTA of a user only); 7.. per round r < 8: codes ready, scored + appended,
shrink done).  python scripts/trace_k6.py /tmp/k6.trace"""
import sys
import numpy as np

raw = open(sys.argv[1], "rb").read()
grid, n = np.frombuffer(raw[:8], np.int32)
t = np.frombuffer(raw[8:], np.int64).reshape(grid, n).astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "phi staged", "S computed", "cluster sync", "chunk scored", "list published", "merged"]
for r in range(4):
    names += [f"r{r} codes ready", f"r{r} scored+appended", f"r{r} shrink done"]
names += ["end: kth found", "end: list written", "merge: floor", "merge: gathered", "merge: sorted",
          "psi pass0 staged", "psi pass0 computed", "psi pass1 staged", "psi pass1 computed", "-", "-"]
print(f"grid {grid}; times in us from the first CTA start (min / median / max over CTAs)")
for i, nm in enumerate(names):
    if nm == "-":
        continue
    v = t[:, i][t[:, i] > 0] - t0
    if len(v):
        print(f"  {i} {nm:16s} {v.min() / 1e3:8.2f} {np.median(v) / 1e3:8.2f} {v.max() / 1e3:8.2f}  (n={len(v)})")
raw_i = np.frombuffer(raw[8:], np.int64).reshape(grid, n)
last = raw_i[:, 6] > 0
print("  merge CTA(s): n3 =", raw_i[last, 31].tolist(), " floor key =", [hex(x & 0xFFFFFFFFFFFFFFFF) for x in raw_i[last, 30].tolist()])
print("  chunk candidates at the end (min/median/max):", int(raw_i[:, 29].min()), int(np.median(raw_i[:, 29])), int(raw_i[:, 29].max()))
