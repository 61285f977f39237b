# ncu --set full captures of the tcgen05 attention (base T=6 ctx 4096, drafter T=1 ctx 600)
tag=${1:-r2attn}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 5 -c 1 \
  -o gpurun_out/${tag}_t6 python tools/one_attn.py 6 64 8 128 4096 1 10 > gpurun_out/${tag}_ncu1.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 5 -c 1 \
  -o gpurun_out/${tag}_t1 python tools/one_attn.py 1 32 8 128 600 1 10 > gpurun_out/${tag}_ncu2.log 2>&1; echo "ncu rc=$?"
