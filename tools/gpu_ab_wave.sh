# batched (fuzzy-group) attention capped to one wave of CTAs: C2 bench A/B vs libespec_ab.so,
# C5 points (lp 4 / 8, gamma 5, ctx 512 / 2K / 8K) for both builds, parity subset
tag=${1:-wave}
mkdir -p gpurun_out
bash tools/gpu_ab_bench.sh $tag 3
for lib in libespec_ab.so libespec_b200.so; do
  echo "== $lib"; ESPEC_LIB=$lib ESPEC_C5_LPS=4,8 ESPEC_C5_NS=5 timeout 900 python tools/sweep_c5.py 512,2048,8192 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: j = json.loads(l)
    except Exception: continue
    print(j)"
done > gpurun_out/${tag}_c5.txt 2>&1; cat gpurun_out/${tag}_c5.txt | cut -c1-300
timeout 900 python -m pytest tests/test_gpu_bf16_shapes.py tests/test_gpu_parity.py tests/test_gpu_stages.py -x -q > gpurun_out/${tag}_tests.txt 2>&1; tail -2 gpurun_out/${tag}_tests.txt
