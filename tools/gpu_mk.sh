mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_megakernel.py -x -q > gpurun_out/r1c_mk.log 2>&1; rc=$?; echo "mk rc=$rc"; tail -30 gpurun_out/r1c_mk.log
if [ $rc -eq 0 ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1c_gpu.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/r1c_gpu.log
timeout 900 python bench.py --no-cpu > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err; echo "bench rc=$?"; cat gpurun_out/r1c_bench.json | head -c 3000; tail -5 gpurun_out/r1c_bench.err
fi
