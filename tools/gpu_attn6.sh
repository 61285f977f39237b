tag=${1:-r2m}
mkdir -p gpurun_out
for d in 0 1 2; do
for spec in "6 64 8 128 4096" "1 32 8 128 600" "6 64 8 128 600"; do set -- $spec
  ESPEC_ATTN_DIAG=$d ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== diag $d T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done; done
