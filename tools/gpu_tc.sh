timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q 2>&1 | tail -2
timeout 300 python tools/bench_tc.py 2>&1 | tail -10
ESPEC_TC_NO_TMA=1 timeout 300 python tools/bench_tc.py 2>&1 | tail -5
