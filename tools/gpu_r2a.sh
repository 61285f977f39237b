mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2a_gpu.log
timeout 1200 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/r2a_bench.json
