timeout 300 python -m pytest tests/test_gpu_megakernel.py -x -q 2>&1 | grep -E "FAILED|passed|failed|timed out|Error" | head -8
ESPEC_MK=0 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k bf16 2>&1 | tail -3
