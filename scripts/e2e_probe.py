"""Host-side cost of one serving query (diagnostics): python bench-like loop of
pq_search with pinned host buffers vs the raw C ABI call with prebuilt
arguments, and the API pieces (workspace query, pointer checks).
    python scripts/e2e_probe.py c2a"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_09992_b200 as pq  # noqa: E402
import pqsynth  # noqa: E402

cfg = pqsynth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2a"]
idx = pq.pq_create(pqsynth.codes(cfg), b=cfg.b)
B, K, d = cfg.B, cfg.K, cfg.d
F_h = torch.from_numpy(pqsynth.phi(cfg)).pin_memory()
P_d = torch.from_numpy(pqsynth.psi(cfg)).cuda()
ids_h = torch.empty((B, K), dtype=torch.int32).pin_memory()
sc_h = torch.empty((B, K), dtype=torch.float32).pin_memory()
L = pq.load_library()
nb = int(L.pq_search_workspace_bytes(idx.handle, B, d, K))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


args = (idx.handle, ctypes.c_void_p(F_h.data_ptr()), ctypes.c_void_p(P_d.data_ptr()), B, d, K, 0,
        ctypes.c_void_p(ws.data_ptr()), nb, ctypes.c_void_p(ids_h.data_ptr()), ctypes.c_void_p(sc_h.data_ptr()),
        ctypes.c_void_p(0), ctypes.c_void_p(st))
print("binding pq_search (pinned host io)  %.1f us" % timeit(lambda: pq.pq_search(idx, F_h, P_d, K, ws=ws, ids=ids_h, scores=sc_h)))
print("raw ctypes pq_search_ex             %.1f us" % timeit(lambda: L.pq_search_ex(*args)))
print("pq_search_workspace_bytes           %.1f us" % timeit(lambda: L.pq_search_workspace_bytes(idx.handle, B, d, K), 5000))
F_d = F_h.cuda()
ids_d = torch.empty((B, K), dtype=torch.int32, device="cuda")
sc_d = torch.empty((B, K), dtype=torch.float32, device="cuda")
args_d = (idx.handle, ctypes.c_void_p(F_d.data_ptr()), ctypes.c_void_p(P_d.data_ptr()), B, d, K, 0,
          ctypes.c_void_p(ws.data_ptr()), nb, ctypes.c_void_p(ids_d.data_ptr()), ctypes.c_void_p(sc_d.data_ptr()),
          ctypes.c_void_p(0), ctypes.c_void_p(st))
print("raw ctypes, device io + sync        %.1f us" % timeit(lambda: (L.pq_search_ex(*args_d), torch.cuda.synchronize())))
print("raw ctypes, device io, no sync      %.1f us" % timeit(lambda: L.pq_search_ex(*args_d)))
e = torch.cuda.Event()
print("empty sync                          %.1f us" % timeit(lambda: torch.cuda.synchronize()))
