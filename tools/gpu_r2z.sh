bash tools/gpu_full.sh r2z
bash tools/gpu_attn.sh r2z
bash tools/gpu_attn_ncu.sh r2z
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py single > gpurun_out/r2z_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|workload done" gpurun_out/r2z_memcheck.log | tail -2
