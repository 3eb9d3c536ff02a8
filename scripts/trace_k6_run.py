"""Run pq_search (K6) on a config with the phase trace on (diagnostics build:
PQTOPK_NVCC_EXTRA=-DK6_TRACE python -m paper_2408_09992_b200.build --force).
    python scripts/trace_k6_run.py c2a gpurun_out/k6_c2a.trace"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_09992_b200 as pq  # noqa: E402
import pqsynth  # noqa: E402

cfg = pqsynth.CONFIGS[sys.argv[1]]
idx = pq.pq_create(pqsynth.codes(cfg), b=cfg.b)
tun = os.environ.get("PQTOPK_TUNING", "")
if tun:
    idx.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in tun.split(",") if kv)})
F = torch.from_numpy(pqsynth.phi(cfg)).cuda()
P = torch.from_numpy(pqsynth.psi(cfg)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
noflush = os.environ.get("TRACE_NOFLUSH") == "1"    # warm-L2 comparison
for i in range(6):
    if not noflush:
        flush.fill_(1)
    if i == 5:
        os.environ["PQTOPK_K6_TRACE"] = sys.argv[2]
    pq.pq_search(idx, F, P, cfg.K)
    torch.cuda.synchronize()
print(idx.search_plan(cfg.B, cfg.d, cfg.K))
