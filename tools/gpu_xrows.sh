timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/gpu_ab.sh ESPEC_X=0 ESPEC_X=1
timeout 600 python tools/sweep_c5.py 512 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if r['lp'] in (1,4) or r['alg']!='easyspec': print(r['alg'], r['n'], r['lp'], round(r['ms_per_iter'],2), round(r['verify_ms'],2), round(r['calibrate_ms'],2), round(r['draft_ms'],2))"
