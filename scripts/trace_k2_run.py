"""Run pq_score_topk (K2 v3) on a config with the CTA trace on (diagnostics build:
PQTOPK_NVCC_EXTRA=-DK2_TRACE python -m paper_2408_09992_b200.build --force).
    python scripts/trace_k2_run.py c2 gpurun_out/k2_c2.trace"""
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
S = pq.pq_subscores(torch.from_numpy(pqsynth.phi(cfg)).cuda(), torch.from_numpy(pqsynth.psi(cfg)).cuda())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(4):
    flush.fill_(1)
    if i == 3:
        os.environ["PQTOPK_K2_TRACE"] = sys.argv[2]
    pq.pq_score_topk(idx, S, cfg.K)
    torch.cuda.synchronize()
print(idx.plan(cfg.B, cfg.K))
