"""Per-source-line warp-stall breakdown of the first kernel in an ncu report.
    python scripts/ncu_lines.py gpurun_out/k6_c7.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in reasons}
lines = []
for r in rows[hi + 1:]:
    if r and r[0]:
        try:
            lines.append((int(r[iS]), r[0], r[1][:70], {c: int(r[idx[c]] or 0) for c in reasons}))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in lines) or 1
lines.sort(key=lambda x: -x[0])
for s, ln, src, d in lines[:N]:
    top = sorted(d.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {ln:>4} {src:70s} " + " ".join(f"{k[6:]}={100 * v / max(s, 1):.0f}%" for k, v in top))
