# ncu --set full captures of the tcgen05 attention on the final build: base T=6 ctx 8192, drafter T=1 ctx 8192
# (ticket combine), drafter T=1 ctx 600 x4 layers (one-wave batched launch)
tag=${1:-r2attn2}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 5 -c 1 \
  -o gpurun_out/${tag}_t6_8k python tools/one_attn.py 6 64 8 128 8192 1 10 > gpurun_out/${tag}_ncu1.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 5 -c 1 \
  -o gpurun_out/${tag}_t1_8k python tools/one_attn.py 1 32 8 128 8192 1 10 > gpurun_out/${tag}_ncu2.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 5 -c 1 \
  -o gpurun_out/${tag}_t1_600x4 python tools/one_attn.py 1 32 8 128 600 4 10 > gpurun_out/${tag}_ncu3.log 2>&1; echo "ncu rc=$?"
for w in 0 1; do echo "== ESPEC_ATTN_WAVE=$w"; ESPEC_ATTN_WAVE=$w timeout 120 python tools/bench_attn.py; done > gpurun_out/${tag}_sweep.txt 2>&1; cat gpurun_out/${tag}_sweep.txt
