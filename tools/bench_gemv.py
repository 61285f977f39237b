"""Isolated decode-GEMV roofline sweep over the C2 shapes (espec_bench_gemv)."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402

SHAPES = {  # name: (K, N, nprob, epi)
    "draft.qkv x3 (fuzzy group)": (4096, 6144, 3, 0), "draft.qkv": (4096, 6144, 1, 0),
    "draft.o": (4096, 4096, 1, 1), "draft.gate_up": (4096, 28672, 1, 2), "draft.down": (14336, 4096, 1, 1),
    "draft.head": (4096, 128256, 1, 0),
    "base.qkv": (8192, 10240, 1, 0), "base.o": (8192, 8192, 1, 1), "base.gate_up": (8192, 57344, 1, 2),
    "base.down": (28672, 8192, 1, 1), "base.head": (8192, 128256, 1, 0),
}


def main():
    L = E.lib()
    L.espec_bench_gemv.argtypes = [C.c_int] * 7 + [C.POINTER(C.c_double)] * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    res = {}
    for name, (K, N, npb, epi) in SHAPES.items():
        us, by = C.c_double(), C.c_double()
        st = L.espec_bench_gemv(K, N, T, npb, epi, 50, 0, C.byref(us), C.byref(by))
        if st != 0:
            print(name, "status", st)
            continue
        gbs = by.value / (us.value * 1e-6) / 1e9
        res[name] = dict(K=K, N=N, nprob=npb, T=T, us=us.value, GBps=gbs, frac=gbs / peak)
        print(f"{name:28s} K={K:6d} N={N:6d} x{npb} T={T:2d}  {us.value:8.1f} us  {gbs:7.0f} GB/s  {gbs / peak:5.1%}")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
