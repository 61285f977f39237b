timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/bench_attn.py 2>&1 | tail -8
bash tools/gpu_ab.sh ESPEC_MK=0 ESPEC_MK=1
