"""tcgen05 prefill GEMM throughput (espec_bench_tc) at the C2 prefill shapes."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_02493_b200 import espec as E  # noqa: E402

SHAPES = [("base.gate_up", 8192, 57344), ("base.down", 28672, 8192), ("base.qkv", 8192, 10240),
          ("draft.gate_up", 4096, 28672), ("draft.head-like", 4096, 32768)]


def main():
    L = E.lib()
    L.espec_bench_tc.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_double)] * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    for M in (128, 256):
        for name, K, N in SHAPES:
            us, fl = C.c_double(), C.c_double()
            st = L.espec_bench_tc(M, K, N, 20, 0, C.byref(us), C.byref(fl))
            if st:
                print(name, "status", st)
                continue
            tf = fl.value / us.value / 1e6
            print(f"M={M:3d} {name:16s} K={K:6d} N={N:6d} {us.value:9.1f} us {tf:7.1f} TFLOP/s ({tf / peak:5.1%} of measured)")


if __name__ == "__main__":
    main()
