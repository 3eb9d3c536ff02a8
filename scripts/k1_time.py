"""Time K1 (pq_subscores) alone for a config: python scripts/k1_time.py c2"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_09992_b200 as pq  # noqa: E402
import pqsynth  # noqa: E402

cfg = pqsynth.CONFIGS[sys.argv[1]]
F = torch.from_numpy(pqsynth.phi(cfg)).cuda()
P = torch.from_numpy(pqsynth.psi(cfg)).cuda()
S = torch.empty((cfg.B, cfg.m, cfg.b), dtype=torch.float32, device="cuda")
for _ in range(3):
    pq.pq_subscores(F, P, S)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
e0.record()
for _ in range(n):
    pq.pq_subscores(F, P, S)
e1.record()
torch.cuda.synchronize()
print(f"{cfg.name} K1 UB={os.environ.get('PQTOPK_K1_UB', 'auto')}: {e0.elapsed_time(e1) / n * 1e3:.1f} us")
