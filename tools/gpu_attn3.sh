tag=${1:-r2j}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "parity or bf16 or megakernel or attn or prefill" > gpurun_out/${tag}_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${tag}_gpu.log
for ppi in 0 2 4 8 16; do
  echo "== ppi $ppi (0 = capacity rule)"; ESPEC_ATTN_PPI=$ppi timeout 300 python tools/bench_attn.py
done > gpurun_out/${tag}_ppi.txt 2>&1
cat gpurun_out/${tag}_ppi.txt
for spec in "6 64 8 128 4096" "1 32 8 128 600"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done
