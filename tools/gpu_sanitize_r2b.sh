# compute-sanitizer memcheck of this round's late changes: the tcgen05 prefill tail (default
# run) and the ticket attention combine (forced, 1-page chunks so every pass splits)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py single \
  > gpurun_out/r2b_san_memcheck_single.log 2>&1; echo "memcheck default rc=$?"; grep -E "ERROR SUMMARY|workload done" gpurun_out/r2b_san_memcheck_single.log | tail -2
ESPEC_ATTN_COMBINE=ticket ESPEC_ATTN_PPI=1 timeout 1500 $CS --tool memcheck --print-limit 20 --error-exitcode 9 \
  python tools/sanitize_workload.py single > gpurun_out/r2b_san_memcheck_ticket.log 2>&1; echo "memcheck ticket rc=$?"
grep -E "ERROR SUMMARY|workload done" gpurun_out/r2b_san_memcheck_ticket.log | tail -2
