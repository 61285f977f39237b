# tcgen05 prefill GEMM: throughput sweep + one ncu --set full capture (base gate/up, M=256)
tag=${1:-r2tc}
mkdir -p gpurun_out
timeout 300 python tools/bench_tc.py > gpurun_out/${tag}_tc.txt 2>&1; cat gpurun_out/${tag}_tc.txt
cat > /tmp/one_tc.py <<'PY'
import ctypes as C, sys, os
sys.path.insert(0, os.getcwd())
from paper_2502_02493_b200 import espec as E
L = E.lib(); L.espec_bench_tc.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_double)] * 2
us, fl = C.c_double(), C.c_double()
print(L.espec_bench_tc(256, 8192, 57344, 3, 0, C.byref(us), C.byref(fl)), us.value)
PY
timeout 600 ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/${tag}_gateup python /tmp/one_tc.py > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"
