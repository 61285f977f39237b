"""Run one paged-attention shape a few times (for an ncu capture).
usage: python tools/one_attn.py T n_heads n_kv dh ctx nprob [iters]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402

T, H, kv, dh, ctx, npb = (int(a) for a in sys.argv[1:7])
iters = int(sys.argv[7]) if len(sys.argv) > 7 else 5
L = E.lib()
L.espec_bench_attn.argtypes = [C.c_int] * 8 + [C.POINTER(C.c_double)] * 2
us, by = C.c_double(), C.c_double()
st = L.espec_bench_attn(T, H, kv, dh, ctx, npb, iters, 0, C.byref(us), C.byref(by))
print(f"status {st}: {us.value:.2f} us")
