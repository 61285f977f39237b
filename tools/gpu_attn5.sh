tag=${1:-r2l}
mkdir -p gpurun_out
timeout 300 python tools/bench_attn.py > gpurun_out/${tag}_attn.txt 2>&1; cat gpurun_out/${tag}_attn.txt
for spec in "6 64 8 128 4096" "1 32 8 128 600"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done
timeout 900 python tools/site_times.py > gpurun_out/${tag}_sites.txt 2>&1; cat gpurun_out/${tag}_sites.txt
