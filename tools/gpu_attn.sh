# decode attention evidence: isolated sweep over C2 shapes, per-CTA timelines,
# pages-per-chunk sweep, in-stream site times -> gpurun_out/<tag>_*
tag=${1:-r2attn}
mkdir -p gpurun_out
timeout 120 python tools/bench_attn.py > gpurun_out/${tag}_attn.txt 2>&1; cat gpurun_out/${tag}_attn.txt
for ppi in 2 4 8 16; do echo "== ppi $ppi"; ESPEC_ATTN_PPI=$ppi timeout 120 python tools/bench_attn.py; done > gpurun_out/${tag}_ppi.txt 2>&1
for spec in "6 64 8 128 4096" "1 32 8 128 600" "6 64 8 128 600"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done > gpurun_out/${tag}_trace.txt 2>&1
timeout 900 python tools/site_times.py > gpurun_out/${tag}_sites.txt 2>&1
