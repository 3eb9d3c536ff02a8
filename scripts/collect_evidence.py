"""Copy one evidence pass (scripts/gpu_evidence_r03.sh, TAG) from gpurun_out/ into profiles/<dir>/ and
refresh profiles/k2_traffic_<cfg>.json (bench.py's roofline.traffic) from the pass's ncu --set full summaries.
    python scripts/collect_evidence.py r03p [r03]"""
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else "r03"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", sub)
os.makedirs(dst, exist_ok=True)

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def bench_line(log):
    lines = [l for l in open(log) if l.startswith("{")]
    return lines[-1] if lines else None


for f in sorted(os.listdir(src)):
    if tag not in f:
        continue
    p = os.path.join(src, f)
    if f.startswith("bench_") and f.endswith(".log"):
        line = bench_line(p)
        name = f[:-4].replace("bench_default_", "bench_c4_").replace("bench_ref_", "bench_ref_c4_")
        if line:
            open(os.path.join(dst, name + ".json"), "w").write(line)
    elif f.endswith("_ncu.txt") or f.startswith("launches_") or f.startswith("smoke_"):
        shutil.copy(p, os.path.join(dst, f))
    elif f.startswith("gpu_tests_"):
        tail = open(p).read().strip().splitlines()[-3:]
        open(os.path.join(dst, f), "w").write("\n".join(tail) + "\n")

# traffic files from the full captures: <kernel>_<cfg>_<tag>_ncu.txt
for f in sorted(os.listdir(src)):
    m = re.match(r"(k\d)_(c\w+?)_%s_ncu\.txt$" % re.escape(tag), f)
    if not m:
        continue
    txt = open(os.path.join(src, f)).read()
    vals = {}
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        mm = re.search(re.escape(key) + r"\s+([0-9.]+)\s+(\w+)", txt)
        if mm:
            vals[key] = float(mm.group(1)) * UNIT[mm.group(2)]
    kn = re.search(r"Kernel Name\s+(.*?)\s*$", txt, re.M)
    if len(vals) == 2:
        out = {"dram_bytes_per_launch": int(vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]),
               "dram_read": int(vals["dram__bytes_read.sum"]), "dram_write": int(vals["dram__bytes_write.sum"]),
               "kernel": kn.group(1) if kn else "", "source": f"ncu --set full, profiles/{sub}/{f}"}
        json.dump(out, open(os.path.join(ROOT, "profiles", f"k2_traffic_{m.group(2)}.json"), "w"), indent=1)
        print(m.group(2), out["dram_bytes_per_launch"])
