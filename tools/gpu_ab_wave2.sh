# one-wave fuzzy attention capped at 8 pages per CTA: C5 points (lp 4 / 8, gamma 5, ctx 512 / 2K / 8K)
# for both builds, then the C2 bench A/B
tag=${1:-wave2}
mkdir -p gpurun_out
for lib in libespec_ab.so libespec_b200.so; do
  echo "== $lib"; ESPEC_LIB=$lib ESPEC_C5_LPS=4,8 ESPEC_C5_NS=5 timeout 900 python tools/sweep_c5.py 512,2048,8192 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: j = json.loads(l)
    except Exception: continue
    if j.get('alg') == 'easyspec': print(j['ctx'], 'lp', j['lp'], 'ms/iter %.2f' % j['ms_per_iter'], 'calib %.2f' % j['calibrate_ms'], 'draft %.2f' % j['draft_ms'], 'verify %.2f' % j['verify_ms'])"
done > gpurun_out/${tag}_c5.txt 2>&1; cat gpurun_out/${tag}_c5.txt
bash tools/gpu_ab_bench.sh $tag 3
