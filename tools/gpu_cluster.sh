# cluster-combine A/B: parity, isolated attention and the C2 bench with the
# chunks combined in a cluster (default) vs the combine kernel
tag=${1:-r2cl}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bf16_shapes.py tests/test_gpu_parity.py tests/test_gpu_stages.py -x -q \
  > gpurun_out/${tag}_tests.txt 2>&1; tail -3 gpurun_out/${tag}_tests.txt
for cl in 0 8 16; do echo "== cluster cap $cl"; ESPEC_ATTN_CLUSTER=$cl timeout 120 python tools/bench_attn.py; done \
  > gpurun_out/${tag}_attn.txt 2>&1; cat gpurun_out/${tag}_attn.txt
for cl in 0 16 0 16; do echo "== cluster cap $cl"; ESPEC_ATTN_CLUSTER=$cl timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu --no-arms 2>/dev/null | tail -1 | cut -c1-400; done \
  > gpurun_out/${tag}_bench.txt 2>&1; cat gpurun_out/${tag}_bench.txt
