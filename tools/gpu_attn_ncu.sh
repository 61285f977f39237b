# ncu full captures of the attention kernel (source-level)
tag=${1:-r2h}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 5 -c 1 \
  -o gpurun_out/${tag}_attn4096 python tools/one_attn.py 6 64 8 128 4096 1 10 > gpurun_out/${tag}_ncu1.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_mma -s 5 -c 1 \
  -o gpurun_out/${tag}_attn600t1 python tools/one_attn.py 1 32 8 128 600 1 10 > gpurun_out/${tag}_ncu2.log 2>&1; echo "ncu rc=$?"
