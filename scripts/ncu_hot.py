"""Top stall lines + per-function sample shares of one kernel in an ncu report.
    python scripts/ncu_hot.py gpurun_out/k2_c4_v3b.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
si = hdr.index("Source"); wi = hdr.index("Warp Stall Sampling (All Samples)"); ei = hdr.index("Instructions Executed")
tot = sum(int(r[wi]) for r in data)
print("total samples", tot)
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][wi]))[:N]:
    print(f"{int(r[wi])/tot*100:5.1f}% {int(r[ei]):>12} {i:5d} {r[si].strip()[:90]}")
acc = 0; start = 0
for i, r in enumerate(data):
    acc += int(r[wi])
    if "RET" in r[si] or "EXIT" in r[si] or i == len(data) - 1:
        if acc: print(f"region {start:5d}-{i:5d} {acc/tot*100:6.2f}%")
        acc = 0; start = i + 1
