"""Read a PQTOPK_K2_TRACE dump (CTA 0 phase timeline of k2_tiled) and print skew / wait stats."""
import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
W, TP = np.frombuffer(raw[:8], np.int32)
a = np.frombuffer(raw[8:], np.int64)
ev = a[:W * TP * 3].reshape(W, TP, 3).astype(np.float64)
iss = a[W * TP * 3:].astype(np.float64)
valid = (ev[:, :, 0] > 0).all(0) & (ev[:, :, 2] > 0).all(0)
n = int(valid.sum())
t0 = ev[:, 0, 0].min()
ev -= t0; iss -= t0
print(f"W={W} phases traced={n}")
print(" ph  wait_start(min..max)   wait_len(mean,max)  end(min..max)   phase_len(mean)")
for g in range(min(n, int(sys.argv[2]) if len(sys.argv) > 2 else 40)):
    ws, we, pe = ev[:, g, 0], ev[:, g, 1], ev[:, g, 2]
    print(f"{g:3d} {ws.min():9.0f}..{ws.max():9.0f}  {np.mean(we-ws):8.0f} {np.max(we-ws):8.0f}  {pe.min():9.0f}..{pe.max():9.0f}  {np.mean(pe-we):8.0f}")
wl = (ev[:, :n, 1] - ev[:, :n, 0]).sum() / (ev[:, :n, 2] - ev[:, :n, 0]).sum()
print(f"fraction of warp time waiting for tables: {wl:.3f}")
sk = (ev[:, :n, 2].max(0) - ev[:, :n, 2].min(0)).mean()
print(f"mean end-of-phase skew (cycles): {sk:.0f}; mean phase length {np.mean(ev[:, :n, 2]-ev[:, :n, 1]):.0f}")
