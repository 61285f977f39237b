# attention: GPU tests, isolated sweep, timelines
tag=${1:-r2g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gpu.log
timeout 300 python tools/bench_attn.py > gpurun_out/${tag}_attn.txt 2>&1; echo "attn rc=$?"; cat gpurun_out/${tag}_attn.txt
for spec in "6 64 8 128 4096" "1 32 8 128 600" "6 64 8 128 600"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done
