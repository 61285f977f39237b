"""Batch-invariance probe: row 0 of a decode GEMV for T = 1..16 rows."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402

L = E.lib()
F = C.POINTER(C.c_float)
L.espec_probe_gemv.argtypes = [C.c_int] * 4 + [F, F, F, C.c_int]
for K, N in ((512, 512), (512, 1536), (1536, 512), (4096, 4096), (8192, 8192), (28672, 8192)):
    rng = np.random.default_rng(K + N)
    x = rng.standard_normal((16, K)).astype(np.float32)
    w = (rng.standard_normal((K, N)) * 0.02).astype(np.float32)
    ref = None
    bad = []
    for T in (1, 2, 8, 9, 12, 16):
        for epi in (0, 1):
            out = np.zeros((T, N), np.float32)
            st = L.espec_probe_gemv(T, K, N, epi, x.ctypes.data_as(F), w.ctypes.data_as(F), out.ctypes.data_as(F), 0)
            assert st == 0, st
            if ref is None:
                ref = out[0].copy()
            if not np.array_equal(out[0], ref):
                bad.append((T, epi, int((out[0] != ref).sum())))
    print(K, N, "row0 identical for all T" if not bad else f"DIFFERS: {bad}")
