for ppi in 1 2 4; do echo "== ppi $ppi"; ESPEC_ATTN_PPI=$ppi timeout 300 python tools/bench_attn.py 2>&1 | head -5; done
bash tools/gpu_ab.sh ESPEC_ATTN_PPI=1 ESPEC_ATTN_PPI=2 ESPEC_ATTN_PPI=1 ESPEC_ATTN_PPI=2
