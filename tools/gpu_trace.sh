timeout 600 python -m pytest tests/test_gpu_megakernel.py -x -q 2>&1 | tail -2
mkdir -p gpurun_out
ESPEC_MK_TRACE=gpurun_out/mktrace timeout 600 python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 > gpurun_out/trace_bench.log 2>&1; echo "trace rc=$?"
ls gpurun_out/ | grep mktrace
for f in gpurun_out/mktrace.*; do echo "== $f"; python tools/mk_trace.py $f 14; done
timeout 300 python tools/bench_attn.py > gpurun_out/bench_attn.log 2>&1; cat gpurun_out/bench_attn.log
