# same-binary A/B of the attention chunk combine (cluster / combine kernel vs the
# in-kernel ticket combine): isolated sweep per mode and ppi, C2 bench, parity subset
tag=${1:-comb}
mkdir -p gpurun_out
for rep in 1 2; do
  for m in "ESPEC_ATTN_COMBINE=" "ESPEC_ATTN_COMBINE=ticket" "ESPEC_ATTN_COMBINE=ticket ESPEC_ATTN_PPI=4"; do
    echo "== $m"; env $m timeout 120 python tools/bench_attn.py
  done
done > gpurun_out/${tag}_attn.txt 2>&1; cat gpurun_out/${tag}_attn.txt
for spec in "6 64 8 128 4096" "1 32 8 128 8192" "6 64 8 128 8192"; do set -- $spec
  ESPEC_ATTN_COMBINE=ticket ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== ticket T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done > gpurun_out/${tag}_trace.txt 2>&1; cat gpurun_out/${tag}_trace.txt
bash tools/gpu_ab_env.sh ${tag} "ESPEC_ATTN_COMBINE=" "ESPEC_ATTN_COMBINE=ticket" 3
timeout 900 python -m pytest tests/test_gpu_bf16_shapes.py -x -q -k "cluster or pool" > gpurun_out/${tag}_tests.txt 2>&1; tail -3 gpurun_out/${tag}_tests.txt
