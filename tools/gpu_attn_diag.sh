# attention diagnostics: per-CTA timelines + one ncu full capture
tag=${1:-r2f}
mkdir -p gpurun_out
for spec in "6 64 8 128 4096" "1 32 8 128 600" "6 64 8 128 600"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 5 -c 1 \
  -o gpurun_out/${tag}_attn4096 python tools/one_attn.py 6 64 8 128 4096 1 10 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"
