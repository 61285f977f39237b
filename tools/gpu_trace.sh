mkdir -p gpurun_out
ESPEC_MK=1 ESPEC_MK_TRACE=gpurun_out/mktrace timeout 600 python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 > gpurun_out/trace_bench.log 2>&1; echo "trace rc=$?"
ls gpurun_out/ | grep mktrace
for f in gpurun_out/mktrace.*; do echo "== $f"; python tools/mk_trace.py $f 14; done
