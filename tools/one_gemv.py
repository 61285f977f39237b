"""Run ONE decode-GEMV shape a few times (for an ncu --set full capture).

usage: python tools/one_gemv.py K N T nprob epi [reps]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402


def main():
    K, N, T, npb, epi = (int(a) for a in sys.argv[1:6])
    reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
    L = E.lib()
    L.espec_bench_gemv.argtypes = [C.c_int] * 7 + [C.POINTER(C.c_double)] * 2
    us, by = C.c_double(), C.c_double()
    st = L.espec_bench_gemv(K, N, T, npb, epi, reps, 0, C.byref(us), C.byref(by))
    print(f"K={K} N={N} T={T} x{npb} epi={epi}: status {st} {us.value:.1f} us {by.value / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
