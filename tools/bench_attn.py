"""Isolated paged-attention latency sweep (espec_bench_attn)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402

CASES = [  # name, T, n_heads, n_kv, dh, ctx, nprob
    ("draft T=1 ctx 600", 1, 32, 8, 128, 600, 1), ("draft T=1 ctx 600 x3", 1, 32, 8, 128, 600, 3),
    ("draft T=1 ctx 600 x4", 1, 32, 8, 128, 600, 4),
    ("draft T=6 ctx 600", 6, 32, 8, 128, 600, 1), ("base T=6 ctx 600", 6, 64, 8, 128, 600, 1),
    ("base T=1 ctx 600", 1, 64, 8, 128, 600, 1), ("base T=6 ctx 4096", 6, 64, 8, 128, 4096, 1),
    ("base T=6 ctx 8192", 6, 64, 8, 128, 8192, 1), ("draft T=1 ctx 8192", 1, 32, 8, 128, 8192, 1),
]


def main():
    L = E.lib()
    L.espec_bench_attn.argtypes = [C.c_int] * 8 + [C.POINTER(C.c_double)] * 2
    for name, T, H, kv, dh, ctx, npb in CASES:
        us, by = C.c_double(), C.c_double()
        st = L.espec_bench_attn(T, H, kv, dh, ctx, npb, 200, 0, C.byref(us), C.byref(by))
        if st:
            print(name, "status", st)
            continue
        print(f"{name:24s} {us.value:8.2f} us  {by.value / us.value / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
