# same-box A/B of the attention kernel: this build vs paper_2502_02493_b200/libespec_ab.so
# (tools/build_ab.sh), isolated sweep twice each, then a parity subset -> gpurun_out/<tag>_*
tag=${1:-ab}
mkdir -p gpurun_out
for lib in libespec_ab.so libespec_b200.so libespec_ab.so libespec_b200.so; do
  echo "== $lib"; ESPEC_LIB=$lib timeout 120 python tools/bench_attn.py
done > gpurun_out/${tag}_attn.txt 2>&1; cat gpurun_out/${tag}_attn.txt
for spec in "6 64 8 128 4096" "1 32 8 128 8192"; do set -- $spec
  ESPEC_ATTN_TRACE="$1,5" timeout 120 python tools/one_attn.py $1 $2 $3 $4 $5 1 10 > /dev/null 2>&1
  echo "== T=$1 H=$2 ctx=$5"; python tools/attn_trace.py gpurun_out/attn_trace.txt
done > gpurun_out/${tag}_trace.txt 2>&1; cat gpurun_out/${tag}_trace.txt
if [ -n "$AB_TESTS" ]; then
  timeout 900 python -m pytest $AB_TESTS -x -q > gpurun_out/${tag}_tests.txt 2>&1; tail -3 gpurun_out/${tag}_tests.txt
fi
