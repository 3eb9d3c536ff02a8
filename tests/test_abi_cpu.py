"""C-ABI library checks that need no GPU: it loads, exports every symbol the
header declares, and rejects invalid arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pqtopk.h")


@pytest.fixture(scope="module")
def L():
    from paper_2408_09992_b200 import build, binding
    build.build()
    return binding.load_library()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pq_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    from paper_2408_09992_b200 import binding
    assert sorted(binding.EXPORTS) == names


def test_nm_exports(L):
    import subprocess
    from paper_2408_09992_b200 import binding
    out = subprocess.check_output(["nm", "-D", "--defined-only", binding.lib_path()], text=True)
    exported = set(re.findall(r" T (pq_\w+)", out))
    assert set(declared_functions()) <= exported


def test_abi_version_and_counter(L):
    assert L.pq_abi_version() == 2
    assert L.pq_launch_count() >= 0


def _err(L):
    return L.pq_last_error().decode()


def test_create_rejects_bad_args(L):
    h = ctypes.c_void_p()
    codes = np.zeros((4, 2), np.uint8)
    p = ctypes.c_void_p(codes.ctypes.data)
    assert L.pq_create(p, 0, 2, 4, 0, None, ctypes.byref(h)) == 1 and "N" in _err(L)
    assert L.pq_create(p, 4, 0, 4, 0, None, ctypes.byref(h)) == 1
    assert L.pq_create(p, 4, 2, 257, 0, None, ctypes.byref(h)) == 1 and "b" in _err(L)
    assert L.pq_create(p, 4, 2, 4, 2**31 - 2, None, ctypes.byref(h)) == 1
    assert L.pq_create(None, 4, 2, 4, 0, None, ctypes.byref(h)) == 1
    assert h.value is None


def test_subscores_rejects_bad_shapes(L):
    assert L.pq_subscores(None, None, 2, 10, 4, 16, None, None) == 1      # d % m != 0
    assert L.pq_subscores(None, None, 0, 8, 4, 16, None, None) == 0       # B = 0: no-op


def test_topk_rejects_null_index_and_big_k(L):
    assert L.pq_score_topk(None, None, 1, 1, None, 0, None, None, None) == 1
    assert L.pq_merge_topk(None, None, 1, 1, 5000, None, 0, None, None, None) == 6
    assert L.pq_merge_topk(None, None, 0, 1, 5, None, 0, None, None, None) == 1
    assert L.pq_topk_workspace_bytes(None, 1, 1) == 0
