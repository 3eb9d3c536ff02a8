"""Per-region warp-stall samples of an ncu report's SASS source page.
    python scripts/ncu_src_regions.py report.ncu-rep [min_samples]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
mins = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
print("total samples", tot, "instructions", len(data))
for i, r in enumerate(data):
    v = int(r[iS]) if r[iS].isdigit() else 0
    if v >= mins:
        print(f"{i:6d} {v:5d} exec={r[iE]:>8s}  {r[1].strip()[:80]}")
