timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_ab.sh ESPEC_SG_ROTATE=0 ESPEC_SG_ROTATE=1 ESPEC_SG_ROTATE=0 ESPEC_SG_ROTATE=1
