# decode-GEMV timelines (see tools/sg_trace.py); args: trace specs
for spec in "$@"; do
ESPEC_SG_TRACE=$spec timeout 600 python bench.py --steps 2 --warmup 3 --no-arms --no-cpu --e2e-tokens 0 > /dev/null 2>&1
echo "== $spec"; python tools/sg_trace.py gpurun_out/sg_trace.txt
done
