"""K2 v3 candidate-insert counts and end-of-tile accounting for a config (PQTOPK_K2_DEBUG
diagnostics; the counters exist only in -DK2_TRACE builds):
    python scripts/k2_inserts.py c5"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_09992_b200 as pq  # noqa: E402
import pqsynth  # noqa: E402

cfg = pqsynth.CONFIGS[sys.argv[1]]
t0 = time.perf_counter()
idx = pq.pq_create(pqsynth.codes(cfg), b=cfg.b)
torch.cuda.synchronize()
print(f"create {time.perf_counter() - t0:.2f} s  layout {idx.layout()}  plan {idx.plan(cfg.B, cfg.K)}", flush=True)
S = pq.pq_subscores(torch.from_numpy(pqsynth.phi(cfg)).cuda(), torch.from_numpy(pqsynth.psi(cfg)).cuda())
pq.pq_score_topk(idx, S, cfg.K)
torch.cuda.synchronize()
os.environ["PQTOPK_K2_DEBUG"] = "1"
pq.pq_score_topk(idx, S, cfg.K)
torch.cuda.synchronize()
