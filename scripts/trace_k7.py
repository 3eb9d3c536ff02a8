"""Summarise a PQTOPK_K6_TRACE dump of the chunk-resident K7 kernel (diagnostics
build, -DK6_TRACE): per-CTA globaltimer stamps.  python scripts/trace_k7.py f"""
import sys
import numpy as np

raw = open(sys.argv[1], "rb").read()
grid, n = np.frombuffer(raw[:8], np.int32)
t = np.frombuffer(raw[8:], np.int64).reshape(grid, n).astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "S share computed", "S reset waited", "S polled + table", "table ready",
         "scored + warp maxima", "candidates", "chunk published", "merge: start (last CTA)",
         "merge: floor", "merge: gathered", "merge: written", "chunk floor",
         "merge: maxima loaded"]
print(f"grid {grid}; times in us from the first CTA start (min / median / max over CTAs)")
for i, nm in enumerate(names):
    v = t[:, i][t[:, i] > 0] - t0
    if len(v):
        print(f"  {i} {nm:24s} {v.min() / 1e3:8.2f} {np.median(v) / 1e3:8.2f} {v.max() / 1e3:8.2f}  (n={len(v)})")
