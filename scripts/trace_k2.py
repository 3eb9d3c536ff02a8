"""Read a PQTOPK_K2_TRACE dump (CTA 0 phase timeline of k2_tiled) and print skew / wait stats.
The library must be built with PQTOPK_NVCC_EXTRA=-DK2_TRACE (python -m paper_2408_09992_b200.build --force)."""
import sys
import numpy as np
raw = open(sys.argv[1], "rb").read()
W, TP = np.frombuffer(raw[:8], np.int32)
a = np.frombuffer(raw[8:], np.int64)
ev = a[:W * TP * 3].reshape(W, TP, 3).astype(np.float64)
units = a[W * TP * 3:W * TP * 3 + TP].reshape(TP // 2, 2).astype(np.float64)
ctas = a[W * TP * 3 + TP:].reshape(-1, 3)
ctas = ctas[ctas[:, 1] > 0]
valid = (ev[:, :, 0] > 0).all(0) & (ev[:, :, 2] > 0).all(0)
n = int(valid.sum())
t0 = ev[:, 0, 0].min()
ev -= t0
print(f"W={W} phases traced={n}")
print(" ph  wait_start(min..max)   wait_len(mean,max)  end(min..max)   phase_len(mean)")
for g in range(min(n, int(sys.argv[2]) if len(sys.argv) > 2 else 40)):
    ws, we, pe = ev[:, g, 0], ev[:, g, 1], ev[:, g, 2]
    print(f"{g:3d} {ws.min():9.0f}..{ws.max():9.0f}  {np.mean(we-ws):8.0f} {np.max(we-ws):8.0f}  {pe.min():9.0f}..{pe.max():9.0f}  {np.mean(pe-we):8.0f}")
wl = (ev[:, :n, 1] - ev[:, :n, 0]).sum() / (ev[:, :n, 2] - ev[:, :n, 0]).sum()
print(f"fraction of warp time waiting for tables: {wl:.3f}")
sk = (ev[:, :n, 2].max(0) - ev[:, :n, 2].min(0)).mean()
print(f"mean end-of-phase skew (cycles): {sk:.0f}; mean phase length {np.mean(ev[:, :n, 2]-ev[:, :n, 1]):.0f}")

nu = int((units[:, 1] > 0).sum())
if nu:
    d = units[:nu, 1] - units[:nu, 0]
    print(f"CTA 0 units: {nu}, cycles per unit mean {d.mean():.0f} min {d.min():.0f} max {d.max():.0f}")
    gaps = units[1:nu, 0] - units[:nu - 1, 1]
    if len(gaps): print(f"  gap between units (cycles) mean {gaps.mean():.0f}")
if len(ctas):
    st, en, tl = ctas[:, 0].astype(np.float64), ctas[:, 1].astype(np.float64), ctas[:, 2]
    t0n = st.min()
    print(f"CTAs: {len(ctas)}; start spread {(st.max()-t0n)/1e3:.1f} us; end min {(en.min()-t0n)/1e6:.3f} ms "
          f"median {(np.median(en)-t0n)/1e6:.3f} max {(en.max()-t0n)/1e6:.3f} ms; tiles/CTA min {tl.min()} max {tl.max()}")
    ns_per_tile = (en - st) / np.maximum(tl, 1)
    print(f"  ns per tile: mean {ns_per_tile.mean():.0f} min {ns_per_tile.min():.0f} max {ns_per_tile.max():.0f}")
# per-warp gaps between a tile's last phase end and the next tile's first wait start
NPh = int(sys.argv[3]) if len(sys.argv) > 3 else 4
if n >= 2 * NPh:
    gaps = []
    for g in range(NPh - 1, n - 1, NPh):
        if g + 1 < n:
            gaps.append((ev[:, g + 1, 0] - ev[:, g, 2]).mean())
    print(f"mean tile-boundary gap per warp (cycles): {np.mean(gaps):.0f}  (NP={NPh})")
    ph_len = [(ev[:, p::NPh, 2] - ev[:, p::NPh, 1])[:, : n // NPh].mean() for p in range(NPh)]
    print("mean phase length by phase:", " ".join(f"{x:.0f}" for x in ph_len))
